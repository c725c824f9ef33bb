"""Parity of the BENCHMARKED configurations with the float64 CPU oracle.

The throughput path (bench.py: CaffeNet, b = 256, TF32, CTA-pair / split-K /
space-to-depth / transposed-fprop GEMM plans that only occur at that size) is
checked at exactly that size, in both precisions, against oracle/refcnn.py
(the reference's algorithm: tensors.py:164-256, problems.py:206-269,
sgd.py:92-112).  The oracle runs its GEMMs through float64 BLAS here
(``refcnn.gemm_impl("blas")``: same products, summation order differing at
the 1e-16 level) so the checker takes seconds, not minutes.

Two views of one training step:

* layer-isolated -- every layer's kernel output is compared with the oracle's
  evaluation of that layer on the GPU's own (fp32, exactly upcast) input, so
  the bound measures that layer's arithmetic, not error carried in from below.
  Max-pool values and argmax indices must be bit-identical (the max of
  identical fp32 values; first-max in (dy, dx) order, problems.py:213-216).
* cascade -- the oracle runs the whole network from the same batch and
  weights; every layer's activation, the loss and every parameter gradient
  are compared (errors compound through 8 layers; argmax flips between fp32
  and fp64 near-ties are counted and reported).

Bounds (normwise relative error; DESIGN.md section 4 states them with the
measured values):

  layer-isolated, forward / data gradient     3xTF32 <= 5e-5   TF32 <= 5e-3
  layer-isolated, weight / bias gradient      3xTF32 <= 3e-4   TF32 <= 5e-3
      (fp32 accumulation over K = b*m^2 = 43,264 .. 774,400 terms)
  max-pool values, argmax indices             bit-identical
  cascade activations                         3xTF32 <= 2e-4   TF32 <= 1e-2
  cascade gradients                           <= 2 sqrt(max activation error)
      (ReLU-mask / argmax flips; see the cascade test)
  g=1 run_sync, 10 steps: W_T                 <= 1e-4 (both)
                          W_T - W_0, V_T      3xTF32 <= 2e-4   TF32 <= 2e-2
"""

import os

import numpy as np
import pytest
import torch

import paper_1606_04487_b200 as P
from paper_1606_04487_b200 import _abi, nets
from paper_1606_04487_b200 import kernels as K
from paper_1606_04487_b200.problems import CNNProblem
from oracle import refcnn as R

pytestmark = pytest.mark.gpu

ISO = {"3xtf32": 5e-5, "tf32": 5e-3}          # forward / data-gradient products, K <= 9216
ISO_RED = {"3xtf32": 3e-4, "tf32": 5e-3}      # weight / bias gradients: K = b*m^2 up to 774,400
CASCADE_ACT = {"3xtf32": 2e-4, "tf32": 1e-2}  # activations through the whole step
CASCADE_GRAD_K = 2.0   # cascade gradients: <= K * sqrt(max activation error), see the cascade test
SYNC_W = 1e-4                                 # run_sync: W_T normwise, both modes
SYNC_DW = {"3xtf32": 2e-4, "tf32": 2e-2}      # run_sync: the learned update W_T - W_0


def nrel(x, ref):
    return float(np.linalg.norm(np.asarray(x) - ref) / max(np.linalg.norm(ref), 1e-300))


def he_weights(net, seed, logit_scale=0.1):
    """N(0, 2/fan_in) weights, 0.1 N(0,1) biases (every layer carries O(1)
    activations at depth), the last layer scaled by ``logit_scale`` so the
    logits are O(1) and the softmax is not saturated (a saturated softmax
    amplifies any logit error into the whole backward); rounded to fp32 so both
    sides see the same W."""
    rng = np.random.default_rng(seed)
    W = np.zeros(net.dim)
    geos = net.geometry()
    last = max(g.index for g in geos if g.param_sizes[0])
    for geo in geos:
        (woff, boff), (wsz, bsz) = geo.param_offsets, geo.param_sizes
        if wsz:
            sc = logit_scale if geo.index == last else 1.0
            W[woff:woff + wsz] = sc * rng.standard_normal(wsz) * np.sqrt(2.0 / (wsz // geo.layer.d_out))
        if bsz:
            W[boff:boff + bsz] = 0.1 * rng.standard_normal(bsz)
    return W.astype(np.float32).astype(np.float64)


def host(act, which="value", b=None):
    """A GpuNet activation (NHWC with channel stride cs, or (b, cs)) as float64 NCHW / (b, f)."""
    t = getattr(act, which)
    t = t if b is None else t[:b]
    if act.spatial:
        return t[..., :act.c].permute(0, 3, 1, 2).double().cpu().numpy()
    return t[:, :act.c].double().cpu().numpy()


def run_step(net, b, precision, W, seed=11):
    """One forward + backward of ``net`` on the GPU at batch b; returns the
    engine (buffers hold every layer's activation and gradient), the batch
    (fp32-exact float64) and the flat gradient."""
    prob = CNNProblem(net, n_examples=b, seed=seed, labels="uniform", precision=precision)
    idx = np.random.default_rng(seed).permutation(b)
    if prob.images is not None:
        X = prob.images[idx].astype(np.float32).astype(np.float64)
        y = prob.labels[idx]
    else:
        it = torch.from_numpy(idx).cuda()
        X = prob.data[it].permute(0, 3, 1, 2).double().cpu().numpy()
        y = prob.data_labels[it].cpu().numpy().astype(np.int64)
    e = prob.engine(b)
    prob.load_batch(e, (X, y))
    Wd = torch.from_numpy(W.astype(np.float32)).cuda()
    e.forward(Wd, b, need_grad=True)
    e.backward(b)
    torch.cuda.synchronize()
    return e, X, y, e.grad.double().cpu().numpy()


# ------------------------------------------------ per-layer oracle pieces --
def conv_fwd_ref(x, Wk, bias, s, p, relu, chunk=32):
    out = np.concatenate([R.conv_lowered(x[i:i + chunk], Wk, s, p) for i in range(0, len(x), chunk)])
    if bias is not None:
        out += bias[None, :, None, None]
    return np.maximum(out, 0.0) if relu else out


def conv_bwd_ref(x, dz, Wk, s, p, need_dx, chunk=32):
    """Weight gradient lower(x)^T dZ summed over images (problems.py:263-267),
    bias gradient, and dX = col2im(dZ K^T) (the extension the oracle adds)."""
    d, c, k, _ = Wk.shape
    b, _, n, _ = x.shape
    m = dz.shape[2]
    gW = np.zeros((c * k * k, d))
    dx = np.empty_like(x) if need_dx else None
    KhT = R.lower_kernel(Wk).T
    for i in range(0, b, chunk):
        j = min(b, i + chunk)
        dR = dz[i:j].transpose(0, 2, 3, 1).reshape(-1, d)
        gW += R.gemm(R.lower(x[i:j], k, s, p).T, dR)
        if need_dx:
            dx[i:j] = R.col2im(R.gemm(dR, KhT), j - i, c, n, k, s, p)
    return gW.T.reshape(Wk.shape), dz.sum(axis=(0, 2, 3)), dx


def layer_views(net, W):
    return R.unpack(net.to_dicts(), net.in_channels, net.in_size, W)


@pytest.fixture(scope="module")
def blas():
    with R.gemm_impl("blas"):
        yield


# ------------------------------------------------------ CaffeNet, b = 256 --
@pytest.mark.slow
@pytest.mark.parametrize("precision", ["3xtf32", "tf32"])
def test_caffenet_b256_layer_isolated(precision, blas):
    """Every kernel of the benchmarked step at the benchmarked size against the
    oracle evaluated on the kernel's own inputs."""
    net = nets.caffenet()
    b = 256
    W = he_weights(net, 5)
    e, X, y, G = run_step(net, b, precision, W)
    views = layer_views(net, W)
    dicts = net.to_dicts()
    geo = {g.index: g for g in net.geometry()}
    gl = {}   # layer index -> op
    li = 0
    for op in e.ops:
        while dicts[li]["kind"] != op.kind:
            li += 1
        gl[li] = op
        li += 1
    bound = ISO[precision]
    report = []
    for li, op in sorted(gl.items()):
        L, pv = dicts[li], views[li]
        x = X if op.inp is e.input else host(op.inp, b=b)
        y_gpu = host(op.out, b=b)
        if op.kind == "conv":
            ref = conv_fwd_ref(x, pv[0], pv[1] if len(pv) > 1 else None, L["stride"], L["pad"], op.relu)
            report.append((li, "conv fwd", nrel(y_gpu, ref), bound))
            dz = host(op.out, "grad", b)
            gW, gb, dx = conv_bwd_ref(x, dz, pv[0], L["stride"], L["pad"], not op.first_param_layer)
            (woff, boff), (wsz, bsz) = geo[li].param_offsets, geo[li].param_sizes
            for name, got, want in (("conv wgrad", G[woff:woff + wsz], gW.ravel()),
                                    ("conv bgrad", G[boff:boff + bsz], gb)):
                report.append((li, name, nrel(got, want), ISO_RED[precision]))
            if dx is not None:
                if op.inp.fused_relu:
                    dx = dx * (x > 0)
                report.append((li, "conv dgrad", nrel(host(op.inp, "grad", b), dx), bound))
        elif op.kind == "pool":
            yr, arg = R._pool_fwd(x, L)
            # (the engine's max pools over a ReLU output mark non-positive windows
            # in the argmax sign bit, omni.h pool mode 2; the index is the low bits)
            ga = op.argmax[: b * op.m * op.m * op.inp.c].view(b, op.m, op.m, op.inp.c) & 0x7FFFFFFF
            ga = ga.permute(0, 3, 1, 2).cpu().numpy()
            report.append((li, "pool values", float(np.abs(y_gpu - yr).max()), 0.0))
            report.append((li, "argmax diffs", float((ga != arg).sum()), 0.0))
            dyp = host(op.out, "grad", b)
            dxr = R._pool_bwd(dyp, x.shape, arg, L)
            if op.inp.fused_relu:
                dxr = dxr * (x > 0)
            # routing identical; fp32 sums of <= 4 overlapping windows
            report.append((li, "pool bwd", nrel(host(op.inp, "grad", b), dxr), 1e-6))
        elif op.kind == "fc":
            flat = x.reshape(b, -1)
            ref = flat @ pv[0] + (pv[1] if len(pv) > 1 else 0.0)
            ref = np.maximum(ref, 0.0) if op.relu else ref
            report.append((li, "fc fwd", nrel(y_gpu, ref), bound))
            dz = host(op.out, "grad", b)
            (woff, boff), (wsz, bsz) = geo[li].param_offsets, geo[li].param_sizes
            report.append((li, "fc wgrad", nrel(G[woff:woff + wsz], (flat.T @ dz).ravel()), ISO_RED[precision]))
            report.append((li, "fc bgrad", nrel(G[boff:boff + bsz], dz.sum(0)), ISO_RED[precision]))
            dflat = dz @ pv[0].T
            if op.inp.fused_relu:
                dflat = dflat * (flat > 0)
            report.append((li, "fc dgrad", nrel(host(op.inp, "grad", b).reshape(b, -1), dflat), bound))
    # softmax-CE (problems.py:221-233, 246-248) on the GPU's logits
    logits = host(e.logits, b=b)
    pr = R.softmax(logits)
    pr[np.arange(b), y] -= 1.0
    report.append(("softmax", "dlogits", nrel(host(e.logits, "grad", b), pr / b), 1e-5))
    loss = float(e.loss_buf.item())
    report.append(("softmax", "loss", abs(loss - R.xent(logits, y)) / max(1.0, abs(loss)), 1e-5))
    print(f"\nCaffeNet b=256 {precision} layer-isolated errors (bound):")
    for li, what, err, bnd in report:
        print(f"  layer {li!s:>7} {what:<12} {err:.3e}  ({bnd:.0e})")
    for li, what, err, bnd in report:
        assert err <= bnd if bnd == 0.0 else err < bnd, (li, what, err, bnd)


def oracle_outputs(net, W, X):
    """The oracle cascade (problems.py:206-219 generalised, as refcnn.forward)
    keeping every layer's OUTPUT and every max-pool's argmax."""
    dicts = net.to_dicts()
    views = layer_views(net, W)
    h, outs, args = X, [], {}
    for li, (L, pv) in enumerate(zip(dicts, views)):
        if L["kind"] == "conv":
            h = conv_fwd_ref(h, pv[0], pv[1] if len(pv) > 1 else None, L["stride"], L["pad"], False)
        elif L["kind"] == "relu":
            h = np.maximum(h, 0.0)
        elif L["kind"] == "pool":
            h, args[li] = R._pool_fwd(h, L)
        else:
            h = h.reshape(h.shape[0], -1) @ pv[0] + (pv[1] if len(pv) > 1 else 0.0)
        outs.append(h)
    return outs, args


@pytest.mark.slow
@pytest.mark.parametrize("precision", ["3xtf32", "tf32"])
def test_caffenet_b256_cascade(precision, blas):
    """The whole step from the same batch and weights: per-layer activations,
    loss and every parameter gradient against the oracle's cascade.

    Activations carry the compounded arithmetic error (bounded absolutely).
    Gradients are discontinuous in the activations: a ReLU mask bit
    (problems.py:261, strict z > 0) or a max-pool argmax (:215-216) flips
    wherever an activation within the forward error of 0 / of a tie sits, and
    each flip moves a whole O(|dZ|) gradient entry.  The flipped fraction grows
    linearly with the activation error e, so the gradient error grows like
    sqrt(e); the bound is CASCADE_GRAD_K * sqrt(max activation error), with the
    flip counts printed.  The per-kernel arithmetic is bounded tightly by the
    layer-isolated test."""
    net = nets.caffenet()
    b = 256
    W = he_weights(net, 5)
    e, X, y, G = run_step(net, b, precision, W)
    dicts = net.to_dicts()
    outs, args = oracle_outputs(net, W, X)
    report, flips, mask_flips = [], {}, {}
    li = 0
    for op in e.ops:
        while dicts[li]["kind"] != op.kind:
            li += 1
        last = li + 1 if op.kind in ("conv", "fc") and op.relu else li   # fused ReLU
        got = host(op.out, b=b).reshape(outs[last].shape)
        report.append((last, f"{op.kind} out", nrel(got, outs[last])))
        if last != li:   # ReLU mask: GPU (post-ReLU > 0) vs oracle (pre-ReLU > 0)
            mask_flips[li] = int(((got > 0) != (outs[li] > 0)).sum())
        if op.kind == "pool" and li in args:
            ga = op.argmax[: b * op.m * op.m * op.inp.c].view(b, op.m, op.m, op.inp.c) & 0x7FFFFFFF
            flips[li] = int((ga.permute(0, 3, 1, 2).cpu().numpy() != args[li]).sum())
        li = last + 1
    logits = outs[-1]
    ref_loss = R.xent(logits, y)
    loss = float(e.loss_buf.item())
    ref_g = R.grad(dicts, net.in_channels, net.in_size, W, X, y)
    greport = []
    for geo in net.geometry():
        for off, sz, nm in zip(geo.param_offsets, geo.param_sizes, ("weight", "bias")):
            if sz:
                greport.append((geo.index, f"{geo.layer.kind} {nm} grad", nrel(G[off:off + sz], ref_g[off:off + sz])))
    act_err = max(err for _, _, err in report)
    gbound = CASCADE_GRAD_K * np.sqrt(act_err)
    print(f"\nCaffeNet b=256 {precision} cascade: loss {loss:.7f} vs {ref_loss:.7f}; max activation error "
          f"{act_err:.2e} -> gradient bound {gbound:.2e}\n  argmax flips per max-pool layer {flips} of "
          f"{ {li: int(a.size) for li, a in args.items()} } windows; ReLU mask flips per layer {mask_flips}")
    for li, what, err in report + greport:
        print(f"  layer {li!s:>3} {what:<16} {err:.3e}")
    assert act_err < CASCADE_ACT[precision], report
    assert abs(loss - ref_loss) < CASCADE_ACT[precision] * max(1.0, ref_loss)
    for _, _, err in greport:
        assert err < gbound, (greport, flips, mask_flips)


# --------------------------------------------- g = 1 multi-step weights ---
@pytest.mark.slow
@pytest.mark.parametrize("name,b", [("lenet", 64), ("cifar10_quick", 128)])
@pytest.mark.parametrize("precision", ["3xtf32", "tf32"])
def test_run_sync_weights_vs_oracle(name, b, precision, blas):
    """run_sync (sgd.py:210-256) for 10 steps at the config's batch size: the
    learned update W_T - W_0 and the sampled loss trace against the oracle's
    run_sync on the same data, seed and hyperparameters."""
    steps, seed, n_ex = 10, 3, 512
    prob = CNNProblem(name, n_examples=n_ex, seed=2, precision=precision)
    net = prob.net
    # the oracle sees the fp32 images the device trains on
    images = prob.images.astype(np.float32).astype(np.float64)
    W0 = prob.initial_weights().astype(np.float32).astype(np.float64)   # 0.01 N(0,1), problems.py:194-195
    hp = P.Hyperparams(eta=0.01, mu=0.9, lam=5e-4, b=b)
    state = P.SGDState.fresh(W0)
    tr = P.run_sync(prob, hp, state, P.StopRule(max_steps=steps), seed=seed)
    Wr, Vr, losses = R.run_sync(net.to_dicts(), net.in_channels, net.in_size, images, prob.labels,
                                W0, hp.eta, hp.mu, hp.lam, b, steps, seed)
    errw = nrel(tr.final_state.W, Wr)
    err = nrel(tr.final_state.W - W0, Wr - W0)
    errv = nrel(tr.final_state.V, Vr)
    print(f"\n{name} b={b} {precision}: W rel err {errw:.3e}, W_T - W_0 rel err {err:.3e}, "
          f"V rel err {errv:.3e}, loss trace max rel err "
          f"{float(np.max(np.abs(tr.losses - losses) / np.abs(losses))):.3e} (final {losses[-1]:.6f})")
    assert errw < SYNC_W
    assert err < SYNC_DW[precision] and errv < SYNC_DW[precision]
    assert np.allclose(tr.losses, losses, rtol=SYNC_DW[precision])


# ------------------------------------------------ argmax with ties -------
@pytest.mark.parametrize("k,s,pad,ceil", [(3, 2, 0, True), (2, 2, 0, True), (3, 2, 1, False), (3, 1, 1, True)])
def test_maxpool_argmax_ties_bit_exact(k, s, pad, ceil):
    """Max pooling on inputs full of exact ties (post-ReLU zeros and repeated
    quantised values): pooled values and argmax indices bit-identical to the
    oracle's first-max routing (problems.py:213-216), and the routed backward
    exact (integer-valued upstream gradients, so every sum is exact)."""
    rng = np.random.default_rng(k * 100 + s * 10 + pad)
    b, c, n = 8, 40, 27
    x = np.maximum(np.round(rng.standard_normal((b, c, n, n)) * 2) / 2, 0.0)   # ~50% zeros, many ties
    x[:, :3] = 0.0                                                              # all-zero channels
    x[:, 3] = 1.5                                                               # all-equal channel
    L = {"kind": "pool", "mode": "max", "k": k, "stride": s, "pad": pad, "ceil": ceil}
    yr, arg = R._pool_fwd(x, L)
    o = yr.shape[2]
    cs = K.round_up(c, 4)
    Xd = torch.zeros((b, n, n, cs), device="cuda")
    Xd[..., :c] = torch.from_numpy(x).permute(0, 2, 3, 1).float().cuda()
    Yd = torch.zeros((b, o, o, cs), device="cuda")
    Ad = torch.zeros(b * o * o * c, dtype=torch.int32, device="cuda")
    K.pool_fwd(0, Xd, c, k, s, pad, ceil, Yd, Ad)
    ga = Ad.view(b, o, o, c).permute(0, 3, 1, 2).cpu().numpy()
    assert np.array_equal(Yd[..., :c].permute(0, 3, 1, 2).double().cpu().numpy(), yr)
    assert np.array_equal(ga, arg), int((ga != arg).sum())
    dy = rng.integers(-3, 4, size=yr.shape).astype(np.float64)
    dxr = R._pool_bwd(dy, x.shape, arg, L)
    dYd = torch.zeros((b, o, o, cs), device="cuda")
    dYd[..., :c] = torch.from_numpy(dy).permute(0, 2, 3, 1).float().cuda()
    dXd = torch.full((b, n, n, cs), 7.0, device="cuda")
    K.pool_bwd(0, dYd, (b, n, n, cs), c, k, s, pad, ceil, Ad, None, 0, dXd)
    assert np.array_equal(dXd[..., :c].permute(0, 3, 1, 2).double().cpu().numpy(), dxr)
    # the ReLU-mask form the engine uses below a fused ReLU (mask from the pooled output)
    K.pool_bwd(0, dYd, (b, n, n, cs), c, k, s, pad, ceil, Ad, Yd, 2, dXd)
    assert np.array_equal(dXd[..., :c].permute(0, 3, 1, 2).double().cpu().numpy(), dxr * (x > 0))
