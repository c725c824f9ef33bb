"""Parity of the B200 path with the reference (golden fixtures) and the CPU oracle.

Tolerances (normwise relative error unless stated), 3xTF32 mode:
  lowering / lifting / argmax-routing           bit-exact
  conv_lowered, gemm                           <= 2e-6
  per-network loss                             <= 1e-5 relative (CaffeNet 5e-5)
  per-network gradient (each parameter tensor) <= 2e-5 (CaffeNet 1e-4)
  g = 1 multi-step weights (8 steps)           <= 1e-4
  g > 1 deterministic schedule                 event log exact, weights <= 1e-4
TF32 mode (the throughput path): gradient <= 5e-2, reported only.
"""

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_1606_04487_b200 as P  # noqa: E402
from paper_1606_04487_b200 import nets  # noqa: E402
from paper_1606_04487_b200.problems import CNNProblem, TinyCNNProblem  # noqa: E402
from oracle import refcnn as R  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    return np.load(os.path.join(GOLD, name))


def nrel(x, ref):
    return float(np.linalg.norm(np.asarray(x) - ref) / max(np.linalg.norm(ref), 1e-300))


# ------------------------------------------------------- operator API ----
def test_lower_lift_bit_exact_vs_reference():
    z = gold("lower.npz")
    i = 0
    while f"case{i}_geom" in z:
        b, c, n, k, s, p, start, b_p = (int(v) for v in z[f"case{i}_geom"])
        spec = P.ConvSpec(n=n, k=k, d_in=c, d_out=1, stride=s, pad=p)
        got = P.lower(P.Tensor4(z[f"case{i}_D"]), spec, b_p=b_p, start=start)
        assert np.array_equal(got.matrix, z[f"case{i}_Dhat"]), i
        i += 1
    spec = P.ConvSpec(n=5, k=3, d_in=2, d_out=3, pad=1)
    R_ = np.random.default_rng(0).standard_normal((2 * 25, 3))
    assert np.array_equal(P.lift(R_, spec, 2).values, R.lift(R_, 2, 5, 3))


def test_conv_gemm_vs_reference():
    z = gold("conv.npz")
    i = 0
    while f"conv{i}_geom" in z:
        n, k, din, dout, s, p, b = (int(v) for v in z[f"conv{i}_geom"])
        spec = P.ConvSpec(n=n, k=k, d_in=din, d_out=dout, stride=s, pad=p)
        for b_p in (1, b):
            got = P.conv_lowered(P.Tensor4(z[f"conv{i}_D"]), P.Tensor4(z[f"conv{i}_K"]), spec, b_p=b_p, workers=2)
            assert nrel(got.values, z[f"conv{i}_R"]) < 2e-6
        i += 1
    kat = P.conv_lowered(P.Tensor4(z["kat_D"]), P.Tensor4(z["kat_K"]), P.ConvSpec(n=3, k=2, d_in=1, d_out=1))
    assert np.allclose(kat.values.reshape(2, 2), [[6, 8], [12, 14]], atol=1e-5)
    assert nrel(P.gemm(z["gemm_A"], z["gemm_B"]), z["gemm_C"]) < 2e-6
    assert np.allclose(P.gemm([[1.0, 2.0], [3.0, 4.0]], [[5.0], [6.0]]), [[17.0], [39.0]], atol=1e-4)


def test_sgd_step_kat():
    s = P.sgd_step(P.SGDState(W=np.array([1.0]), V=np.array([0.0])), P.Hyperparams(eta=0.1, mu=0.9),
                   np.array([2.0]), np.array([1.0]))
    assert abs(s.V[0] + 0.2) < 1e-7 and abs(s.W[0] - 0.8) < 1e-7 and s.t == 1


# ----------------------------------------------------------- TinyCNN -----
@pytest.mark.parametrize("tag", ["s8c4", "s16c10"])
def test_tiny_cnn_vs_reference(tag):
    z = gold("tinycnn.npz")
    size, classes, n_ex, b, seed = (int(v) for v in z[f"{tag}_meta"])
    prob = TinyCNNProblem(size, classes, seed=seed, n_examples=n_ex)
    assert np.array_equal(prob.images, z[f"{tag}_images"]) and np.array_equal(prob.labels, z[f"{tag}_labels"])
    W0 = prob.initial_weights()
    assert np.array_equal(W0, z[f"{tag}_W0"])
    batch = prob.sample_batch(P.batch_stream(seed), b)
    X, y = batch
    assert np.array_equal(X, z[f"{tag}_bx"])
    g = prob.grad(W0, batch)
    assert nrel(g, z[f"{tag}_grad"]) < 2e-5
    assert abs(prob.loss(W0, batch) - float(z[f"{tag}_loss"])) < 1e-5 * abs(float(z[f"{tag}_loss"]))
    assert abs(prob.full_loss(W0) - float(z[f"{tag}_full_loss"])) < 1e-5
    g2 = prob.grad(W0, (X, y))  # host-array batch, the reference's batch type
    assert nrel(g2, g) < 1e-6


def test_run_sync_vs_reference():
    z = gold("tinycnn.npz")
    eta, mu, lam, b, steps, seed = z["sync_hp"]
    prob = TinyCNNProblem(8, 4, seed=3, n_examples=64)
    hp = P.Hyperparams(eta=float(eta), mu=float(mu), lam=float(lam), b=int(b))
    tr = P.run_sync(prob, hp, prob.initial_state(), P.StopRule(max_steps=int(steps)), seed=int(seed))
    assert nrel(tr.final_state.W, z["sync_W"]) < 1e-4
    assert nrel(tr.final_state.V, z["sync_V"]) < 1e-3
    assert np.allclose(tr.losses, z["sync_losses"], rtol=1e-5)


def test_simulate_deterministic_vs_reference():
    z = gold("tinycnn.npz")
    prob = TinyCNNProblem(8, 4, seed=3, n_examples=64)
    hp = P.Hyperparams(eta=0.05, mu=0.9, lam=1e-3, b=16)
    cfg = P.SimConfig(plan=P.ExecutionPlan(N=8, g=4), profile=P.PhaseProfile(T_cc=8.0, T_nc=0.1, t_fc=0.5),
                      hp=hp, problem=prob, max_updates=12, seed=5)
    tr = P.simulate(cfg)
    ev = np.array([[e.group_id, e.read_step, e.write_step, e.staleness] for e in tr.events])
    assert np.array_equal(ev, z["sim_events"][:, :4])
    assert nrel(tr.final_state.W, z["sim_W"]) < 1e-4
    st = P.staleness_stats(tr, burn_in=4)
    assert st.mean == 3.0


@pytest.mark.parametrize("g", [2, 4])
def test_implicit_momentum_estimator_vs_reference(g):
    """simulator.py:244-321 on the device: trajectories in HBM, float64 run sums,
    device full gradients, 2x2 normal equations -- vs the reference's own
    estimate on the same seeded runs (fp32 state: the fitted coefficient agrees
    to ~1e-3 of its scale)."""
    z = gold("implicit_momentum.npz")
    prob = TinyCNNProblem(8, 4, seed=3, n_examples=64)
    hp = P.Hyperparams(eta=0.05, mu=0.0, lam=0.0, b=8)
    cfg = P.SimConfig(plan=P.ExecutionPlan(N=4, g=g), profile=P.PhaseProfile(T_cc=4.0, T_nc=0.0, t_fc=0.01),
                      hp=hp, problem=prob, service_mode="exponential", max_updates=80, seed=3)
    a = P.estimate_implicit_momentum(cfg, n_runs=8)
    ref = float(z[f"im_g{g}"])
    print(f"g={g}: device {a:.6f} reference {ref:.6f}")
    assert abs(a - ref) < 5e-3


# ------------------------------------------------ networks vs oracle ------
# (net, batch, gradient tol, loss tol): fp32 accumulation error grows with depth and
# fan-in (CaffeNet: K up to 9216 through 8 layers), so its bound is looser.
NETS = [("lenet", 6, 2e-5, 1e-5), ("cifar10_quick", 4, 2e-5, 1e-5), ("caffenet", 2, 1e-4, 5e-5)]


def scaled_weights(net, seed):
    """N(0, 2/fan_in) weights (He scaling) so every layer of a deep net carries
    O(1) activations and the comparison is not dominated by saturation."""
    rng = np.random.default_rng(seed)
    W = np.zeros(net.dim)
    for geo in net.geometry():
        woff, boff = geo.param_offsets
        wsz, bsz = geo.param_sizes
        if wsz:
            fan_in = wsz // geo.layer.d_out
            W[woff:woff + wsz] = rng.standard_normal(wsz) * np.sqrt(2.0 / fan_in)
        if bsz:
            W[boff:boff + bsz] = 0.1 * rng.standard_normal(bsz)
    return W


def argmax_flips(engine, net, W, X, b):
    """Per max-pool layer index: how many windows picked a different argmax on the
    GPU than in the float64 oracle, for the same inputs."""
    _, cache = R.forward(net.to_dicts(), net.in_channels, net.in_size, W, X)
    ref_args = [data[1] for kind, data in cache if kind == "pool"]
    geo_pools = [g.index for g in net.geometry() if g.layer.kind == "pool"]
    out = {}
    gpu_pools = [op for op in engine.ops if op.kind == "pool"]
    for li, op, ra in zip(geo_pools, gpu_pools, ref_args):
        if ra is None:
            continue
        o, c = op.m, op.inp.c
        ga = op.argmax[: b * o * o * c].view(b, o, o, c).permute(0, 3, 1, 2).cpu().numpy()
        out[li] = int((ga != ra).sum())
    return out


def per_param_errors(net, g, ref):
    errs = []
    for geo in net.geometry():
        for off, sz in zip(geo.param_offsets, geo.param_sizes):
            if sz and off >= 0:
                errs.append((geo.layer.kind, geo.index, nrel(g[off:off + sz], ref[off:off + sz])))
    return errs


@pytest.mark.parametrize("name,b,gtol,ltol", NETS)
def test_network_grad_vs_oracle(name, b, gtol, ltol):
    net = nets.get(name)
    prob = CNNProblem(net, n_examples=max(16, b), seed=1, precision="3xtf32")
    W = scaled_weights(net, seed=7)
    batch = prob.sample_batch(P.batch_stream(2), b)
    if prob.images is not None:
        X, y = batch
    else:
        idx = torch.from_numpy(batch.idx).cuda()
        X = prob.data[idx].permute(0, 3, 1, 2).double().cpu().numpy()
        y = prob.data_labels[idx].cpu().numpy()
    ref = R.grad(net.to_dicts(), net.in_channels, net.in_size, W, X, y, workers=os.cpu_count() or 1)
    ref_loss = R.loss(net.to_dicts(), net.in_channels, net.in_size, W, X, y)
    g = prob.grad(W, batch)
    flips = argmax_flips(prob.engine(b), net, W, X, b)
    loss = prob.loss(W, batch)
    assert abs(loss - ref_loss) <= ltol * max(1.0, abs(ref_loss)), (loss, ref_loss)
    errs = per_param_errors(net, g, ref)
    # A max-pool near-tie that fp32 and fp64 resolve differently re-routes the
    # gradient of one window to another pixel (problems.py:215-216); only the
    # conv layers below that pool see it, as a local O(1/sqrt(n)) perturbation.
    first_flip = min((li for li, nf in flips.items() if nf), default=None)
    for kind, li, e in errs:
        bound = 5e-3 if first_flip is not None and li < first_flip else gtol
        assert e < bound, (kind, li, e, flips, errs)
    # tf32 (throughput) mode, reported with a loose bound
    p32 = CNNProblem(net, n_examples=max(16, b), seed=1, precision="tf32")
    g32 = p32.grad(W, batch)
    assert nrel(g32, ref) < 5e-2


def test_full_grad_and_chunked_loss():
    prob = CNNProblem("lenet", n_examples=300, seed=4)
    W = prob.initial_weights()
    net = prob.net
    ref = R.grad(net.to_dicts(), 1, 28, W, prob.images, prob.labels, workers=os.cpu_count() or 1)
    assert nrel(prob.full_grad(W), ref) < 2e-5
    ref_loss = R.loss(net.to_dicts(), 1, 28, W, prob.images, prob.labels)
    assert abs(prob.full_loss(W) - ref_loss) < 1e-5


def test_sgd_step_bit_exact_vs_oracle():
    """The drop-in sgd_step (float64 K8) equals the reference's NumPy update
    (sgd.py:92-101) bit for bit, stale regulariser snapshot included."""
    rng = np.random.default_rng(4)
    n = 100_003
    W, V, g, wr = (rng.standard_normal(n) for _ in range(4))
    hp = P.Hyperparams(eta=0.0123, mu=0.87, lam=3e-4)
    s = P.sgd_step(P.SGDState(W=W, V=V, t=5), hp, g, wr)
    W2, V2 = R.sgd_step(W, V, g, wr, hp.eta, hp.mu, hp.lam)
    assert np.array_equal(s.V, V2) and np.array_equal(s.W, W2) and s.t == 6


@pytest.mark.parametrize("g", [1, 2, 4, 8])
def test_measured_he_deterministic(g):
    """measured_he (simulator.py:216-223) after a 100-event burn-in is within
    2% of he_predict for deterministic services (SPEC measured_he examples);
    g = 1 is exactly t_conv(N) + t_fc; the N = 8, g = 8 profile of the SPEC
    example is FC-saturated at t_fc."""
    prob = TinyCNNProblem(8, 4, seed=3, n_examples=64)
    plan = P.ExecutionPlan(N=8, g=g)
    prof = P.PhaseProfile(T_cc=10.0, T_nc=0.1, t_fc=2.0)
    cfg = P.SimConfig(plan=plan, profile=prof, hp=P.Hyperparams(eta=0.01, mu=0.5, b=8), problem=prob,
                      max_updates=300, seed=1)
    tr = P.simulate(cfg)
    he = P.measured_he(tr, burn_in=100)
    pred = P.he_predict(plan, prof)
    if g == 1:
        assert abs(he - (P.t_conv(8, prof) + prof.t_fc)) < 1e-9
    if g == 8:
        assert P.fc_saturated(plan, prof) and abs(he - 2.0) < 1e-9
    assert abs(he - pred) <= 0.02 * pred, (g, he, pred)


@pytest.mark.parametrize("T_cc,t_fc", [(2.0, 2.0), (10.0, 0.01)])
def test_measured_he_exponential(T_cc, t_fc):
    """Exponential services, 10k events: within 10% of he_predict (SPEC) --
    away from the saturation boundary, where queueing (which the closed form
    ignores) is negligible: deeply FC-saturated (he = t_fc) and deeply
    conv-bound (he = (t_conv + t_fc) / g)."""
    prob = TinyCNNProblem(8, 4, seed=3, n_examples=64)
    plan = P.ExecutionPlan(N=8, g=4)
    prof = P.PhaseProfile(T_cc=T_cc, T_nc=0.1, t_fc=t_fc)
    cfg = P.SimConfig(plan=plan, profile=prof, hp=P.Hyperparams(eta=0.001, mu=0.0, b=4), problem=prob,
                      service_mode="exponential", max_updates=10_000, loss_sample_interval=10_000, seed=2)
    tr = P.simulate(cfg)
    he, pred = P.measured_he(tr, burn_in=100), P.he_predict(plan, prof)
    assert abs(he - pred) <= 0.10 * pred, (he, pred)
