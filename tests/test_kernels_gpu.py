"""GPU unit tests of the individual sm_100a kernels through the C-ABI.

Floating-point kernels are compared against a plain PyTorch fp64 reference of
the same op (normwise relative error; 3xTF32 bound 5e-6 * max(1, sqrt(K/1000)):
tf32 hi/lo products lose ~2^-21 and the tensor-core fp32 accumulation is not
IEEE-exact); data-movement kernels must be bit-exact.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_1606_04487_b200 import _abi, kernels as K  # noqa: E402

DEV = "cuda"


def rel_err(x, ref):
    x = x.double()
    ref = ref.double()
    return float((x - ref).norm() / max(ref.norm().item(), 1e-300))


def make_operand(rows_i, rows_r, mn_major, gen):
    """Return (storage tensor, ld, logical (i x r) fp64 matrix)."""
    logical = torch.randn(rows_i, rows_r, generator=gen, dtype=torch.float64)
    if mn_major:
        ld = K.round_up(rows_i, 4)
        st = torch.zeros(rows_r, ld, dtype=torch.float32)
        st[:, :rows_i] = logical.t().float()
    else:
        ld = K.round_up(rows_r, 4)
        st = torch.zeros(rows_i, ld, dtype=torch.float32)
        st[:, :rows_r] = logical.float()
    return st.to(DEV), ld, logical.float().double()


SHAPES = [
    (128, 128, 32),
    (300, 96, 363),
    (257, 200, 100),
    (1000, 256, 2400),
    (64, 384, 1152),
    (96, 363, 20000),  # few tiles: split-K
    (4, 10, 9),
]


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("prec", ["tf32", "3xtf32"])
def test_gemm_vs_torch(a_mn, b_mn, shape, prec):
    M, N, Kd = shape
    gen = torch.Generator().manual_seed(M * 7 + N * 13 + Kd)
    A, lda, Al = make_operand(M, Kd, a_mn, gen)
    B, ldb, Bl = make_operand(N, Kd, b_mn, gen)
    C = torch.full((M, N), float("nan"), device=DEV)
    K.gemm(M, N, Kd, A, lda, a_mn, B, ldb, b_mn, C, N, precision=_abi.PRECISIONS[prec])
    torch.cuda.synchronize()
    ref = Al @ Bl.t()
    err = rel_err(C.cpu(), ref)
    # fp32 accumulation error grows like sqrt(K)
    tol = 3e-3 if prec == "tf32" else 5e-6 * max(1.0, (Kd / 1000.0) ** 0.5)
    assert err < tol, (shape, a_mn, b_mn, prec, err)


@pytest.mark.parametrize("epi", ["bias", "bias_relu", "relu", "mask", "accum"])
def test_gemm_epilogues(epi):
    M, N, Kd = 333, 130, 250
    gen = torch.Generator().manual_seed(5)
    A, lda, Al = make_operand(M, Kd, False, gen)
    B, ldb, Bl = make_operand(N, Kd, False, gen)
    bias = torch.randn(N, generator=gen).to(DEV)
    aux = torch.randn(M, N, generator=gen).to(DEV)
    C0 = torch.randn(M, N, generator=gen).to(DEV)
    C = C0.clone()
    code = {"bias": _abi.EPI_BIAS, "bias_relu": _abi.EPI_BIAS_RELU, "relu": _abi.EPI_RELU,
            "mask": _abi.EPI_MASK_AUX, "accum": _abi.EPI_ACCUM}[epi]
    K.gemm(M, N, Kd, A, lda, False, B, ldb, False, C, N, precision=_abi.PREC_3XTF32,
           epilogue=code, bias=bias, aux=aux, ld_aux=N)
    torch.cuda.synchronize()
    acc = Al @ Bl.t()
    b64 = bias.cpu().double()
    ref = {"bias": acc + b64, "bias_relu": (acc + b64).clamp_min(0), "relu": acc.clamp_min(0),
           "mask": acc * (aux.cpu().double() > 0), "accum": C0.cpu().double() + acc}[epi]
    assert rel_err(C.cpu(), ref) < 2e-6


@pytest.mark.parametrize("epi", ["bias_relu", "mask"])
def test_gemm_epilogue_operands_read_in_bounds(epi):
    """Small-M GEMM whose bias/aux operands end exactly at the end of a
    segment-sized allocation: the TMA-store epilogue computes whole 32x32
    sub-tiles (128 rows per tile), so any read of rows >= M or columns >= N
    would land past the segment (regression: LeNet FC dgrad, M = 16)."""
    M, N, Kd = 16, 40, 64
    gen = torch.Generator().manual_seed(9)
    A, lda, Al = make_operand(M, Kd, False, gen)
    B, ldb, Bl = make_operand(N, Kd, False, gen)
    seg = 8 << 20   # 32 MiB of fp32: a dedicated, 2 MiB-rounded cudaMalloc segment
    big = torch.empty(seg, device=DEV)
    aux = big[seg - M * N:].view(M, N)
    aux.copy_(torch.randn(M, N, generator=gen).to(DEV))
    big2 = torch.empty(seg, device=DEV)
    bias = big2[seg - N:]
    bias.copy_(torch.randn(N, generator=gen).to(DEV))
    C = torch.empty(M, N, device=DEV)
    code = _abi.EPI_BIAS_RELU if epi == "bias_relu" else _abi.EPI_MASK_AUX
    K.gemm(M, N, Kd, A, lda, False, B, ldb, False, C, N, precision=_abi.PREC_3XTF32,
           epilogue=code, bias=bias, aux=aux, ld_aux=N)
    torch.cuda.synchronize()
    acc = Al @ Bl.t()
    ref = (acc + bias.cpu().double()).clamp_min(0) if epi == "bias_relu" else \
        acc * (aux.cpu().double() > 0)
    assert rel_err(C.cpu(), ref) < 2e-6


def test_gemm_operand_extent_checked():
    A = torch.zeros(8, 8, device=DEV)
    C = torch.zeros(8, 8, device=DEV)
    with pytest.raises(ValueError, match="extent"):
        K.gemm(16, 8, 8, A, 8, False, A, 8, False, C, 8)   # A holds 8 rows, not 16


def test_gemm_simt_reference():
    M, N, Kd = 70, 50, 40
    gen = torch.Generator().manual_seed(1)
    A, lda, Al = make_operand(M, Kd, True, gen)
    B, ldb, Bl = make_operand(N, Kd, False, gen)
    C = torch.empty(M, N, device=DEV)
    K.gemm(M, N, Kd, A, lda, True, B, ldb, False, C, N, precision=_abi.PREC_FP32_SIMT)
    torch.cuda.synchronize()
    assert rel_err(C.cpu(), Al @ Bl.t()) < 1e-6


def test_gemm_bad_args_raise():
    A = torch.zeros(8, 8, device=DEV)
    with pytest.raises(ValueError):
        K.gemm(8, 8, 8, A, 6, False, A, 8, False, A, 8)  # lda not a multiple of 4
    with pytest.raises(ValueError):
        K.gemm(0, 8, 8, A, 8, False, A, 8, False, A, 8)


def ref_lower_np(D, k, s, p):
    """Independent numpy lowering in the reference's (c, kx, ky) column order."""
    b, c, n, _ = D.shape
    m = (n + 2 * p - k) // s + 1
    Dp = np.pad(D, ((0, 0), (0, 0), (p, p), (p, p)))
    out = np.empty((b, m, m, c, k, k), D.dtype)
    for kx in range(k):
        for ky in range(k):
            out[:, :, :, :, kx, ky] = Dp[:, :, kx:kx + s * (m - 1) + 1:s,
                                         ky:ky + s * (m - 1) + 1:s].transpose(0, 2, 3, 1)
    return out.reshape(b * m * m, c * k * k)


@pytest.mark.parametrize("geom", [(2, 3, 9, 3, 1, 1), (3, 1, 8, 3, 1, 1), (2, 3, 27, 11, 4, 0),
                                  (1, 5, 13, 5, 2, 2), (4, 2, 6, 1, 1, 0)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_lower_nchw_bit_exact(geom, dtype):
    b, c, n, k, s, p = geom
    rng = np.random.default_rng(0)
    D = rng.standard_normal((b, c, n, n)).astype(np.float32).astype(np.float64)
    Dt = torch.from_numpy(D).to(dtype).to(DEV)
    got = K.lower_nchw(Dt, k, s, p, 0, b).cpu().numpy()
    want = ref_lower_np(D, k, s, p).astype(got.dtype)
    assert np.array_equal(got, want)
    # padded ld: pad columns are zero
    ld = K.round_up(c * k * k, 4) + 4
    got2 = K.lower_nchw(Dt, k, s, p, 0, b, ld=ld).cpu().numpy()
    assert np.array_equal(got2[:, : c * k * k], want) and not got2[:, c * k * k:].any()


@pytest.mark.parametrize("geom", [(2, 3, 9, 3, 1, 1), (2, 8, 10, 3, 1, 1), (2, 3, 27, 11, 4, 0),
                                  (1, 16, 13, 5, 2, 2)])
def test_lower_nhwc_tap_major_and_col2im_adjoint(geom):
    b, c, n, k, s, p = geom
    rng = np.random.default_rng(1)
    D = rng.standard_normal((b, c, n, n)).astype(np.float32)
    cs = K.round_up(c, 4)
    X = torch.zeros(b, n, n, cs)
    X[..., :c] = torch.from_numpy(D).permute(0, 2, 3, 1)
    Kc = c * k * k
    ld = K.round_up(Kc, 4)
    got = K.lower_nhwc(X.to(DEV), c, k, s, p, ld).cpu().numpy()
    ref = ref_lower_np(D, k, s, p)  # (c, kx, ky) order
    m = (n + 2 * p - k) // s + 1
    ref_tap = ref.reshape(b * m * m, c, k * k).transpose(0, 2, 1).reshape(b * m * m, Kc)
    assert np.array_equal(got[:, :Kc], ref_tap)
    assert not got[:, Kc:].any()
    # adjoint: <lower(X), G> == <X, col2im(G)>
    G = torch.randn(b * m * m, ld, dtype=torch.float32)
    G[:, Kc:] = 0
    dX = torch.zeros(b, n, n, cs, device=DEV)
    K.col2im_nhwc(G.to(DEV), ld, b, n, c, cs, k, s, p, dX)
    lhs = float((torch.from_numpy(got).double() * G.double()).sum())
    rhs = float((X.double() * dX.cpu().double()).sum())
    assert abs(lhs - rhs) <= 1e-4 * max(1.0, abs(lhs))


def test_lift_bit_exact():
    b, m, d = 3, 5, 7
    R = torch.randn(b * m * m, d, dtype=torch.float64)
    got = K.lift_nchw(R.to(DEV), b, m, d).cpu()
    want = R.reshape(b, m, m, d).permute(0, 3, 1, 2)
    assert torch.equal(got, want)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("geom", [(2, 8, 8, 3, 2, 2, 0, True), (2, 55, 55, 5, 3, 2, 0, True),
                                  (3, 32, 32, 4, 3, 2, 0, True), (1, 7, 7, 4, 3, 2, 1, True),
                                  # stride-2 blocked backward: k=4 with odd pad has 3 covering
                                  # windows per axis (must take the per-pixel kernel)
                                  (2, 9, 9, 8, 4, 2, 1, True), (2, 8, 8, 8, 4, 2, 0, False),
                                  (2, 9, 9, 8, 3, 2, 1, False), (2, 8, 8, 8, 2, 2, 0, False)])
def test_pool_fwd_bwd(mode, geom):
    b, h, w, c, k, s, p, ceil_mode = geom
    gen = torch.Generator().manual_seed(3)
    X = torch.randn(b, h, w, c, generator=gen)
    oh = K.pool_out_size(h, k, s, p, ceil_mode)
    ow = K.pool_out_size(w, k, s, p, ceil_mode)
    Y = torch.empty(b, oh, ow, c, device=DEV)
    am = torch.empty(b * oh * ow * c, dtype=torch.int32, device=DEV)
    K.pool_fwd(mode, X.to(DEV), c, k, s, p, ceil_mode, Y, am if mode == 0 else None)
    # reference via explicit loops
    Yr = torch.empty(b, oh, ow, c, dtype=torch.float64)
    for oy in range(oh):
        for ox in range(ow):
            hs, ws = oy * s - p, ox * s - p
            he, we = min(hs + k, h + p), min(ws + k, w + p)
            size = (he - hs) * (we - ws)
            hs, ws, he, we = max(hs, 0), max(ws, 0), min(he, h), min(we, w)
            win = X[:, hs:he, ws:we, :].double()
            Yr[:, oy, ox] = win.amax(dim=(1, 2)) if mode == 0 else win.sum(dim=(1, 2)) / size
    assert torch.allclose(Y.cpu().double(), Yr, rtol=1e-6, atol=1e-6)
    # backward vs autograd of the same reference
    Xa = X.double().requires_grad_(True)
    outs = []
    for oy in range(oh):
        row = []
        for ox in range(ow):
            hs, ws = oy * s - p, ox * s - p
            he, we = min(hs + k, h + p), min(ws + k, w + p)
            size = (he - hs) * (we - ws)
            hs, ws, he, we = max(hs, 0), max(ws, 0), min(he, h), min(we, w)
            win = Xa[:, hs:he, ws:we, :]
            row.append(win.amax(dim=(1, 2)) if mode == 0 else win.sum(dim=(1, 2)) / size)
        outs.append(torch.stack(row, 1))
    Yg = torch.stack(outs, 1)
    dY = torch.randn(b, oh, ow, c, generator=gen)
    Yg.backward(dY.double())
    dX = torch.empty(b, h, w, c, device=DEV)
    K.pool_bwd(mode, dY.to(DEV), X.shape, c, k, s, p, ceil_mode, am if mode == 0 else None,
               None, False, dX)
    assert torch.allclose(dX.cpu().double(), Xa.grad, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("geom", [(2, 55, 55, 96, 3, 2, 0, True), (2, 13, 13, 20, 2, 2, 0, True),
                                  (2, 9, 9, 8, 3, 2, 1, False), (1, 7, 7, 3, 3, 3, 1, True)])
def test_maxpool_bwd_output_mask_equals_input_mask(geom):
    """relu_mask_x = 2 (mask by the pooled output) is bit-identical to masking
    the routed gradient by the ReLU'd input: the routed element is the max."""
    b, h, w, c, k, s, p, ceil_mode = geom
    gen = torch.Generator().manual_seed(21)
    X = torch.randn(b, h, w, c, generator=gen).clamp_min(0).to(DEV)   # post-ReLU (many zeros)
    oh, ow = K.pool_out_size(h, k, s, p, ceil_mode), K.pool_out_size(w, k, s, p, ceil_mode)
    Y = torch.empty(b, oh, ow, c, device=DEV)
    am = torch.empty(b * oh * ow * c, dtype=torch.int32, device=DEV)
    K.pool_fwd(0, X, c, k, s, p, ceil_mode, Y, am)
    dY = torch.randn(b, oh, ow, c, generator=gen).to(DEV)
    d1, d2 = torch.empty_like(X), torch.empty_like(X)
    K.pool_bwd(0, dY, X.shape, c, k, s, p, ceil_mode, am, X, 1, d1)
    K.pool_bwd(0, dY, X.shape, c, k, s, p, ceil_mode, am, Y, 2, d2)
    torch.cuda.synchronize()
    assert torch.equal(d1.cpu(), d2.cpu())


@pytest.mark.parametrize("geom", [(2, 55, 55, 96, 3, 2, 0, True), (2, 13, 13, 20, 2, 2, 0, True),
                                  (2, 9, 9, 8, 3, 2, 1, False), (1, 7, 7, 3, 3, 3, 1, True)])
def test_maxpool_marked_argmax_equals_output_mask(geom):
    """Forward mode 2 (argmax sign bit set where the window max is not > 0) +
    backward without a mask == mode 0 + the relu_mask_x = 2 backward, bit for
    bit; argmax & 0x7fffffff == mode 0's argmax; pooled values identical."""
    b, h, w, c, k, s, p, ceil_mode = geom
    gen = torch.Generator().manual_seed(23)
    X = torch.randn(b, h, w, c, generator=gen).clamp_min(0).to(DEV)
    X[0, : h // 2] = 0.0                                   # whole windows of zeros
    oh, ow = K.pool_out_size(h, k, s, p, ceil_mode), K.pool_out_size(w, k, s, p, ceil_mode)
    Y0, Y2 = torch.empty(b, oh, ow, c, device=DEV), torch.empty(b, oh, ow, c, device=DEV)
    a0 = torch.empty(b * oh * ow * c, dtype=torch.int32, device=DEV)
    a2 = torch.empty_like(a0)
    K.pool_fwd(0, X, c, k, s, p, ceil_mode, Y0, a0)
    K.pool_fwd(2, X, c, k, s, p, ceil_mode, Y2, a2)
    dY = torch.randn(b, oh, ow, c, generator=gen).to(DEV)
    d0, d2 = torch.empty_like(X), torch.empty_like(X)
    K.pool_bwd(0, dY, X.shape, c, k, s, p, ceil_mode, a0, Y0, 2, d0)
    K.pool_bwd(0, dY, X.shape, c, k, s, p, ceil_mode, a2, None, 0, d2)
    torch.cuda.synchronize()
    assert torch.equal(Y0, Y2) and torch.equal(a2 & 0x7FFFFFFF, a0)
    assert bool((a2 < 0).any()) and torch.equal(a2 < 0, ~(Y0.view(-1) > 0))
    assert torch.equal(d0, d2)


def test_softmax_xent():
    b, C = 37, 1000
    gen = torch.Generator().manual_seed(2)
    Z = torch.randn(b, C, generator=gen) * 3
    y = torch.randint(0, C, (b,), generator=gen, dtype=torch.int32)
    loss = torch.empty(1, device=DEV)
    dZ = torch.empty(b, C, device=DEV)
    K.softmax_xent(Z.to(DEV), C, y.to(DEV), b, C, loss, dZ, C, 1.0 / b)
    Zd = Z.double().requires_grad_(True)
    ref = torch.nn.functional.cross_entropy(Zd, y.long())
    ref.backward()
    assert abs(loss.item() - ref.item()) < 1e-5 * abs(ref.item())
    assert rel_err(dZ.cpu(), Zd.grad) < 1e-5


def test_bias_grad_sgd_gather_transpose():
    gen = torch.Generator().manual_seed(4)
    M, N = 10007, 96
    dY = torch.randn(M, N, generator=gen)
    db = torch.empty(N, device=DEV)
    ws = torch.empty(K.bias_grad_ws_elems(M, N), device=DEV)
    K.bias_grad(dY.to(DEV), N, M, N, db, ws)
    assert rel_err(db.cpu(), dY.double().sum(0)) < 1e-6
    n = 1001
    W, V, g, wr = (torch.randn(n, generator=gen) for _ in range(4))
    Wd, Vd = W.to(DEV), V.to(DEV)
    K.sgd_momentum(Wd, Vd, g.to(DEV), wr.to(DEV), 0.1, 0.9, 0.01)
    Vr = 0.9 * V.double() - 0.1 * (g.double() + 0.01 * wr.double())
    assert rel_err(Vd.cpu(), Vr) < 1e-6 and rel_err(Wd.cpu(), W.double() + Vr) < 1e-6
    src = torch.randn(50, 3, 5, 5, generator=gen)
    idx = torch.tensor([3, 3, 49, 0, 7], dtype=torch.int64)
    dst = torch.empty(5, 3, 5, 5, device=DEV)
    K.gather_rows(src.to(DEV), idx.to(DEV), dst)
    assert torch.equal(dst.cpu(), src[idx])
    T = torch.randn(4, 33, 65, generator=gen)
    out = torch.empty(4, 65, 33, device=DEV)
    K.transpose(T.to(DEV), 65, 33 * 65, 33, 65, out, 33, 65 * 33, 4)
    assert torch.equal(out.cpu(), T.transpose(1, 2))


@pytest.mark.parametrize("g,k,n,off", [(1, 2, 4096, 0), (2, 2, 1003, 0), (4, 1, 4096, 1), (2, 4, 777, 3)])
def test_group_updates_equals_eager_rounds(g, k, n, off):
    """One group_updates kernel == the eager round (clone + add_ of the members'
    rows in order, K8, snapshot copy), bit for bit, on vector and scalar paths
    (off > 0: shards at unaligned offsets, as the layer-aligned runtime slices)."""
    gen = torch.Generator().manual_seed(7 + g * k)
    N = g * k
    rows = torch.randn(N, (n + off + 7) // 4 * 4, generator=gen).to(DEV)     # pitch % 4 == 0
    W0, V0 = (torch.randn(n + off, generator=gen).to(DEV) for _ in range(2))
    S0 = [torch.randn(n + off, generator=gen).to(DEV) for _ in range(g)]
    members = [list(range(i * k, i * k + k))[::-1] for i in range(g)]       # any order: summed as listed
    eta, mu, lam = 0.05, 0.9, 1e-3
    W, V, S = W0.clone(), V0.clone(), [s.clone() for s in S0]
    K.group_updates(rows[:, off:], members, W[off:], V[off:], [s[off:] for s in S], eta, mu, lam)
    We, Ve, Se = W0.clone()[off:], V0.clone()[off:], [s.clone()[off:] for s in S0]
    for i in range(g):
        Gi = rows[members[i][0], off:off + n].clone()
        for m in members[i][1:]:
            Gi.add_(rows[m, off:off + n])
        K.sgd_momentum(We, Ve, Gi.contiguous(), Se[i], eta, mu, lam)
        Se[i].copy_(We)
    torch.cuda.synchronize()
    assert torch.equal(W[off:], We) and torch.equal(V[off:], Ve)
    assert all(torch.equal(s[off:], e) for s, e in zip(S, Se))
    assert torch.equal(W[:off], W0[:off])


@pytest.mark.parametrize("rows,cols,lds,ldd", [(36, 256, 256, 36), (256, 36, 36, 260), (49, 50, 52, 49),
                                             (9, 1000, 1000, 12)])
def test_transpose_batched_strided(rows, cols, lds, ldd):
    """Batched transposes of the shapes the engine uses (the pool5 -> fc6
    flatten and its gradient, 36 x 256 per image) and ragged ones: exact,
    strided rows on both sides, nothing written outside the transposed block."""
    gen = torch.Generator().manual_seed(rows * cols)
    batch = 70
    sb, db = rows * lds + 3, cols * ldd + 5
    src = torch.randn(batch * sb, generator=gen)
    dst = torch.full((batch * db,), float("nan"), device=DEV)
    K.transpose(src.to(DEV), lds, sb, rows, cols, dst, ldd, db, batch)
    torch.cuda.synchronize()
    S = torch.as_strided(src, (batch, rows, cols), (sb, lds, 1))
    D = torch.as_strided(dst.cpu(), (batch, cols, rows), (db, ldd, 1))
    assert torch.equal(D, S.transpose(1, 2))
    written = torch.zeros(batch * db, dtype=torch.bool)
    torch.as_strided(written, (batch, cols, rows), (db, ldd, 1)).fill_(True)
    assert torch.isnan(dst.cpu()[~written]).all()


@pytest.mark.parametrize("o,c,k", [(7, 3, 5), (96, 3, 11), (256, 96, 5), (384, 256, 3), (512, 512, 3),
                                   (50, 20, 5)])
def test_conv_weight_tap_roundtrip(o, c, k):
    gen = torch.Generator().manual_seed(o + c + k)
    W = torch.randn(o, c, k, k, generator=gen)
    bias = torch.randn(o, generator=gen)
    ld = K.round_up(c * k * k + 1, 32)
    Wt = torch.full((o, ld), float("nan"), device=DEV)
    K.conv_weight_to_tap(W.to(DEV), o, c, k, Wt, ld, bias=bias.to(DEV))
    ref = W.permute(0, 2, 3, 1).reshape(o, k * k * c)
    got = Wt.cpu()
    assert torch.equal(got[:, : c * k * k], ref)
    assert torch.equal(got[:, c * k * k], bias)
    assert (got[:, c * k * k + 1:] == 0).all()                       # row padding zeroed
    back = torch.empty(o, c, k, k, device=DEV)
    bb = torch.empty(o, device=DEV)
    K.conv_weight_to_tap(back, o, c, k, Wt, ld, inverse=True, bias=bb)
    assert torch.equal(back.cpu(), W) and torch.equal(bb.cpu(), bias)


@pytest.mark.parametrize("o,c,k", [(96, 256, 5), (384, 256, 3), (256, 384, 3), (50, 20, 5), (70, 33, 11)])
def test_conv_weight_flip_layout(o, c, k):
    """Wf[ch*ld + (kx*k + ky)*o + oo] = W[oo, ch, k-1-kx, k-1-ky], zero row padding."""
    gen = torch.Generator().manual_seed(o * c + k)
    W = torch.randn(o, c, k, k, generator=gen)
    ld = K.round_up(o * k * k, 32) + 32
    Wf = torch.full((c, ld), float("nan"), device=DEV)
    K.conv_weight_flip(W.to(DEV), o, c, k, Wf, ld)
    ref = W.flip(2, 3).permute(1, 2, 3, 0).reshape(c, k * k * o)
    got = Wf.cpu()
    assert torch.equal(got[:, : o * k * k], ref)
    assert (got[:, o * k * k:] == 0).all()


@pytest.mark.parametrize("geom", [(2, 3, 27, 11, 4, 0), (2, 8, 10, 3, 1, 1), (1, 5, 9, 3, 1, 1)])
def test_bias_ones_column(geom):
    """The bias rides in the GEMM: Dhat column c*k*k is 1.0 and the staged weights
    carry the bias there; the inverse staging returns the bias (gradient)."""
    b, c, n, k, s, p = geom
    Kc = c * k * k
    ld = K.round_up(Kc + 1, 4)
    X = torch.randn(b, n, n, c, device=DEV)
    D = K.lower_nhwc(X, c, k, s, p, ld, ones_col=True)
    assert torch.all(D[:, Kc] == 1.0) and not D[:, Kc + 1:].any()
    ref = K.lower_nhwc(X, c, k, s, p, K.round_up(Kc, 4))
    assert torch.equal(D[:, :Kc], ref[:, :Kc])
    o = 6
    W = torch.randn(o, c, k, k, device=DEV)
    bias = torch.randn(o, device=DEV)
    Wt = torch.empty(o, ld, device=DEV)
    K.conv_weight_to_tap(W, o, c, k, Wt, ld, bias=bias)
    assert torch.equal(Wt[:, Kc], bias)
    W2 = torch.empty_like(W)
    b2 = torch.empty_like(bias)
    K.conv_weight_to_tap(W2, o, c, k, Wt, ld, inverse=True, bias=b2)
    assert torch.equal(W2, W) and torch.equal(b2, bias)


IMPLICIT_GEOMS = [  # b, n, c, k, s, p, d_out
    (2, 27, 96, 5, 1, 2, 256),
    (3, 13, 64, 3, 1, 1, 96),
    (2, 15, 32, 3, 2, 1, 64),
    (1, 9, 32, 1, 1, 0, 32),
    (2, 13, 384, 3, 1, 1, 256),
]


def _conv_inputs(b, n, c, k, d, seed):
    gen = torch.Generator().manual_seed(seed)
    X = torch.randn(b, n, n, c, generator=gen)
    W = torch.randn(d, c, k, k, generator=gen) / (c * k * k) ** 0.5
    return X.to(DEV), W.to(DEV)


@pytest.mark.parametrize("geom", IMPLICIT_GEOMS)
@pytest.mark.parametrize("prec", ["tf32", "3xtf32"])
def test_conv_implicit_fprop(geom, prec):
    """TMA-im2col implicit GEMM == explicit lowering + GEMM (same operands, same
    K order) and == torch conv2d in float64 within the precision's bound."""
    b, n, c, k, s, p, d = geom
    X, W = _conv_inputs(b, n, c, k, d, 11)
    m = (n + 2 * p - k) // s + 1
    Kc = c * k * k
    ld = K.round_up(Kc, 32)
    Wt = torch.zeros(d, ld, device=DEV)
    K.conv_weight_to_tap(W, d, c, k, Wt, ld)
    pr = _abi.PRECISIONS[prec]
    Y = torch.full((b * m * m, d), float("nan"), device=DEV)
    K.conv_implicit(_abi.CONV_FPROP, X, c, k, s, p, d, Wt, ld, Y, d, precision=pr)
    D = K.lower_nhwc(X, c, k, s, p, ld)
    Yr = torch.empty(b * m * m, d, device=DEV)
    K.gemm(b * m * m, d, Kc, D, ld, False, Wt, ld, False, Yr, d, precision=pr)
    torch.cuda.synchronize()
    assert rel_err(Y.cpu(), Yr.cpu()) < 2e-6, rel_err(Y.cpu(), Yr.cpu())
    ref = torch.nn.functional.conv2d(X.permute(0, 3, 1, 2).double().cpu(), W.double().cpu(),
                                     stride=s, padding=p).permute(0, 2, 3, 1).reshape(b * m * m, d)
    assert rel_err(Y.cpu(), ref) < (3e-3 if prec == "tf32" else 5e-6 * max(1.0, (Kc / 1000) ** 0.5))


@pytest.mark.parametrize("geom", IMPLICIT_GEOMS + [(8, 13, 384, 3, 1, 1, 384)])
@pytest.mark.parametrize("prec", ["tf32", "3xtf32"])
def test_conv_implicit_wgrad(geom, prec):
    """TF32 runs on CTA pairs (M = taps*c > 128: 256-row tiles, half of dY per
    CTA); 3xTF32 on single CTAs."""
    b, n, c, k, s, p, d = geom
    X, _ = _conv_inputs(b, n, c, k, d, 12)
    m = (n + 2 * p - k) // s + 1
    Kc = c * k * k
    ld = K.round_up(Kc, 32)
    dY = torch.randn(b * m * m, d, device=DEV)
    dW = torch.full((d, ld), float("nan"), device=DEV)
    K.conv_implicit(_abi.CONV_WGRAD, X, c, k, s, p, d, dY, d, dW, ld,
                    precision=_abi.PRECISIONS[prec])
    D = K.lower_nhwc(X, c, k, s, p, ld)
    ref = (dY.double().t() @ D[:, :Kc].double()).cpu()
    torch.cuda.synchronize()
    tol = 3e-3 if prec == "tf32" else 5e-6 * max(1.0, (b * m * m / 1000) ** 0.5)
    assert rel_err(dW[:, :Kc].cpu(), ref) < tol


@pytest.mark.parametrize("geom", IMPLICIT_GEOMS + [(8, 13, 384, 3, 1, 1, 256)])
@pytest.mark.parametrize("prec", ["tf32", "3xtf32"])
def test_conv_implicit_wgrad_bias_row(geom, prec):
    """OMNI_CONV_WGRAD_BIAS: the weight gradient plus the bias gradient (column
    sums of dY) in column k*k*c, from one GEMM with a ones operand chunk."""
    b, n, c, k, s, p, d = geom
    X, _ = _conv_inputs(b, n, c, k, d, 14)
    m = (n + 2 * p - k) // s + 1
    Kc = c * k * k
    ld = K.round_up(Kc + 1, 32)
    dY = torch.randn(b * m * m, d, device=DEV)
    dW = torch.full((d, ld), float("nan"), device=DEV)
    pr = _abi.PRECISIONS[prec]
    ws = torch.empty(max(1, K.conv_implicit_workspace_bytes(pr, _abi.CONV_WGRAD_BIAS, b, n, c, k,
                                                            s, p, d)) // 4, device=DEV)
    ws.fill_(float("nan"))   # the ones tile must be written by the call itself
    K.conv_implicit(_abi.CONV_WGRAD_BIAS, X, c, k, s, p, d, dY, d, dW, ld, precision=pr,
                    workspace=ws)
    D = K.lower_nhwc(X, c, k, s, p, K.round_up(Kc, 32))
    ref = (dY.double().t() @ D[:, :Kc].double()).cpu()
    torch.cuda.synchronize()
    tol = 3e-3 if prec == "tf32" else 5e-6 * max(1.0, (b * m * m / 1000) ** 0.5)
    assert rel_err(dW[:, :Kc].cpu(), ref) < tol
    assert rel_err(dW[:, Kc].cpu(), dY.double().sum(0).cpu()) < tol


def test_conv_weight_s2d_inverse_bias_column():
    o, c, k, s = 8, 3, 11, 4
    k2, cp = -(-k // s), K.round_up(s * s * c, 32)
    ld = K.round_up(k2 * k2 * cp + 1, 32)
    Wt = torch.randn(o, ld, device=DEV)
    W = torch.empty(o * c * k * k, device=DEV)
    bias = torch.empty(o, device=DEV)
    K.conv_weight_s2d(W, o, c, k, s, cp, Wt, ld, inverse=True, bias=bias)
    torch.cuda.synchronize()
    assert torch.equal(bias.cpu(), Wt[:, k2 * k2 * cp].cpu())


@pytest.mark.parametrize("geom", [g for g in IMPLICIT_GEOMS if g[4] == 1 and g[6] % 32 == 0])
def test_conv_implicit_dgrad_via_flipped_weights(geom):
    """Stride-1 data gradient as one implicit forward conv of dY with the flipped,
    transposed kernel (padding k-1-p) == col2im of the explicit dgrad GEMM."""
    b, n, c, k, s, p, d = geom
    X, W = _conv_inputs(b, n, c, k, d, 13)
    m = n + 2 * p - k + 1
    dY = torch.randn(b, m, m, d, device=DEV)
    ldf = K.round_up(d * k * k, 32)
    Wf = torch.zeros(c, ldf, device=DEV)
    K.conv_weight_flip(W, d, c, k, Wf, ldf)
    dX = torch.full((b, n, n, c), float("nan"), device=DEV)
    K.conv_implicit(_abi.CONV_FPROP, dY, d, k, 1, k - 1 - p, c, Wf, ldf, dX.view(-1, c), c,
                    precision=_abi.PREC_3XTF32)
    Xd = X.permute(0, 3, 1, 2).double().cpu().requires_grad_(True)
    out = torch.nn.functional.conv2d(Xd, W.double().cpu(), padding=p)
    out.backward(dY.permute(0, 3, 1, 2).double().cpu())
    torch.cuda.synchronize()
    assert rel_err(dX.cpu(), Xd.grad.permute(0, 2, 3, 1)) < 5e-6 * max(1.0, (d * k * k / 1000) ** 0.5)


@pytest.mark.parametrize("b,n,c,s,cp", [(3, 227, 3, 4, 48), (2, 227, 3, 4, 64), (2, 30, 4, 2, 16),
                                         (2, 16, 5, 2, 32), (1, 9, 3, 4, 48)])
def test_space_to_depth_exact(b, n, c, s, cp):
    """Y[img, X, Y, (dx*s + dy)*c + ch] = X[img, s*X + dx, s*Y + dy, ch], zero past
    the image and in the padded channels -- bit-exact against a torch re-layout
    (staged and unstaged kernels; the gathered form with a permuted batch)."""
    gen = torch.Generator().manual_seed(5 + n)
    X = torch.randn(b, n, n, c, generator=gen)
    n2 = -(-n // s)
    Xp = torch.zeros(b, n2 * s, n2 * s, c)
    Xp[:, :n, :n] = X
    ref = Xp.view(b, n2, s, n2, s, c).permute(0, 1, 3, 2, 4, 5).reshape(b, n2, n2, s * s * c)
    want = torch.zeros(b, n2, n2, cp)
    want[..., :s * s * c] = ref
    Y = torch.full((b, n2, n2, cp), float("nan"), device=DEV)
    K.space_to_depth(X.to(DEV), c, s, Y)
    idx = torch.arange(b - 1, -1, -1, dtype=torch.int64)
    Yg = torch.full((b, n2, n2, cp), float("nan"), device=DEV)
    K.space_to_depth_gather(X.to(DEV), idx.to(DEV), c, s, Yg)
    torch.cuda.synchronize()
    assert torch.equal(Y.cpu(), want)
    assert torch.equal(Yg.cpu(), want[idx])


@pytest.mark.parametrize("geom", [(2, 27, 3, 11, 4, 0, 96), (2, 227, 3, 11, 4, 0, 96), (3, 16, 5, 4, 2, 0, 32)])
def test_space_to_depth_conv_equals_strided_conv(geom):
    """A stride-s k x k conv == the stride-1 ceil(k/s)^2 implicit conv of the
    space-to-depth input with the mapped weights; and the weight-gradient maps back."""
    b, n, c, k, s, p, d = geom
    m = (n + 2 * p - k) // s + 1
    gen = torch.Generator().manual_seed(21)
    X = torch.randn(b, n, n, c, generator=gen).to(DEV)
    W = (torch.randn(d, c, k, k, generator=gen) / (c * k * k) ** 0.5).to(DEV)
    k2, n2 = -(-k // s), -(-n // s)
    cp = K.round_up(s * s * c, 32)
    assert n2 - k2 + 1 == m
    Y = torch.empty(b, n2, n2, cp, device=DEV)
    K.space_to_depth(X, c, s, Y)
    ld = K.round_up(k2 * k2 * cp, 32)
    Wt = torch.empty(d, ld, device=DEV)
    K.conv_weight_s2d(W, d, c, k, s, cp, Wt, ld)
    out = torch.empty(b * m * m, d, device=DEV)
    K.conv_implicit(_abi.CONV_FPROP, Y, cp, k2, 1, 0, d, Wt, ld, out, d, precision=_abi.PREC_3XTF32)
    Xd = X.permute(0, 3, 1, 2).double().cpu().requires_grad_(False)
    Wd = W.double().cpu().requires_grad_(True)
    ref = torch.nn.functional.conv2d(Xd, Wd, stride=s)
    torch.cuda.synchronize()
    assert rel_err(out.cpu(), ref.permute(0, 2, 3, 1).reshape(-1, d)) < 5e-6 * max(1.0, (k2 * k2 * cp / 1000) ** 0.5)
    dY = torch.randn(b * m * m, d, generator=gen)
    ref.backward(dY.reshape(b, m, m, d).permute(0, 3, 1, 2).double())
    dWt = torch.empty(d, ld, device=DEV)
    K.conv_implicit(_abi.CONV_WGRAD, Y, cp, k2, 1, 0, d, dY.to(DEV), d, dWt, ld, precision=_abi.PREC_3XTF32)
    dW = torch.empty(d, c, k, k, device=DEV)
    K.conv_weight_s2d(dW, d, c, k, s, cp, dWt, ld, inverse=True)
    torch.cuda.synchronize()
    assert rel_err(dW.cpu(), Wd.grad) < 5e-6 * max(1.0, (b * m * m / 1000) ** 0.5)


@pytest.mark.parametrize("epi", ["store", "bias_relu", "mask"])
def test_conv_implicit_fprop_transposed_form(epi, monkeypatch):
    """Few output channels and many pixels select the C^T = W im2col^T form
    (im2col as the K-major B operand, transposed epilogue); it must equal the
    standard form, epilogues included (bias by row, mask read transposed)."""
    b, n, c, k, s, p, d = 32, 27, 96, 5, 1, 2, 96
    X, W = _conv_inputs(b, n, c, k, d, 31)
    m = n
    ld = K.round_up(c * k * k, 32)
    Wt = torch.zeros(d, ld, device=DEV)
    K.conv_weight_to_tap(W, d, c, k, Wt, ld)
    bias = torch.randn(d, device=DEV)
    aux = torch.randn(b * m * m, d, device=DEV)
    code = {"store": _abi.EPI_STORE, "bias_relu": _abi.EPI_BIAS_RELU, "mask": _abi.EPI_MASK_AUX}[epi]
    outs = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("OMNI_NO_TRANSPOSED_FPROP", env)
        Y = torch.full((b * m * m, d), float("nan"), device=DEV)
        K.conv_implicit(_abi.CONV_FPROP, X, c, k, s, p, d, Wt, ld, Y, d, precision=_abi.PREC_3XTF32,
                        epilogue=code, bias=bias, aux=aux, ld_aux=d)
        torch.cuda.synchronize()
        outs.append(Y.cpu())
    # (the env switch is read once per process, so the second call may still be
    # transposed; compare both against torch instead)
    ref = torch.nn.functional.conv2d(X.permute(0, 3, 1, 2).double().cpu(), W.double().cpu(),
                                     padding=p).permute(0, 2, 3, 1).reshape(-1, d)
    if epi == "bias_relu":
        ref = (ref + bias.double().cpu()).clamp_min(0)
    elif epi == "mask":
        ref = ref * (aux.double().cpu() > 0)
    for Y in outs:
        assert rel_err(Y, ref) < 5e-6 * max(1.0, (c * k * k / 1000) ** 0.5)


def test_space_to_depth_gather_equals_gather_then_transform():
    gen = torch.Generator().manual_seed(43)
    data = torch.randn(20, 27, 27, 3, generator=gen).to(DEV)
    idx = torch.tensor([5, 0, 19, 5, 7], dtype=torch.int64, device=DEV)
    s, n2, cp = 4, 7, 64
    Y1 = torch.full((5, n2, n2, cp), float("nan"), device=DEV)
    Y2 = torch.full((5, n2, n2, cp), float("nan"), device=DEV)
    K.space_to_depth_gather(data, idx, 3, s, Y1)
    K.space_to_depth(data[idx], 3, s, Y2)
    torch.cuda.synchronize()
    assert torch.equal(Y1.cpu(), Y2.cpu())


def test_space_to_depth_conv1_large_batch():
    """CaffeNet conv1 geometry at a batch where the implicit GEMM spans all SMs."""
    b, n, c, k, s, d = 8, 227, 3, 11, 4, 96
    gen = torch.Generator().manual_seed(41)
    X = torch.randn(b, n, n, c, generator=gen).to(DEV)
    W = (torch.randn(d, c, k, k, generator=gen) / (c * k * k) ** 0.5).to(DEV)
    m = (n - k) // s + 1
    k2, n2, cp = 3, 57, 64
    Y = torch.empty(b, n2, n2, cp, device=DEV)
    K.space_to_depth(X, c, s, Y)
    ld = K.round_up(k2 * k2 * cp, 32)
    Wt = torch.empty(d, ld, device=DEV)
    K.conv_weight_s2d(W, d, c, k, s, cp, Wt, ld)
    out = torch.empty(b * m * m, d, device=DEV)
    K.conv_implicit(_abi.CONV_FPROP, Y, cp, k2, 1, 0, d, Wt, ld, out, d, precision=_abi.PREC_3XTF32)
    ref = torch.nn.functional.conv2d(X.permute(0, 3, 1, 2).double().cpu(), W.double().cpu(), stride=s)
    torch.cuda.synchronize()
    assert rel_err(out.cpu(), ref.permute(0, 2, 3, 1).reshape(-1, d)) < 5e-6


def _s2d_conv1(b, gen, n=227, c=3, k=11, s=4, d=96):
    X = torch.randn(b, n, n, c, generator=gen).to(DEV)
    W = (torch.randn(d, c, k, k, generator=gen) / (c * k * k) ** 0.5).to(DEV)
    k2, n2, cp = -(-k // s), -(-n // s), 48
    # 16 floats of slack after the image: the window wgrad's overlapping-row view
    buf = torch.full((b * n2 * n2 * cp + 16,), float("nan"), device=DEV)
    Y = buf[:b * n2 * n2 * cp].view(b, n2, n2, cp)
    K.space_to_depth(X, c, s, Y)
    return X, W, Y, k2, n2, cp


@pytest.mark.parametrize("b,epi", [(1, "bias_relu"), (3, "store"), (20, "bias_relu")])
def test_conv_window_fprop_vs_torch(b, epi):
    """The window implicit GEMM (all 9 taps of a tile read from one staged input
    window by shifted descriptors; weights resident; CTA pairs) == the strided
    11x11 conv, TF32 tolerance; junk (padded-width) rows never written."""
    gen = torch.Generator().manual_seed(60 + b)
    X, W, Xs, k2, n2, cp = _s2d_conv1(b, gen)
    d, m = 96, n2 - k2 + 1
    ld = K.round_up(k2 * k2 * cp, 32)
    Wt = torch.zeros(d, ld, device=DEV)
    K.conv_weight_s2d(W, d, 3, 11, 4, cp, Wt, ld)
    bias = torch.randn(d, generator=gen).to(DEV)
    cs = 100   # a pixel stride wider than d_out: the gap must stay untouched
    out = torch.full((b * m * m, cs), float("nan"), device=DEV)
    code = {"store": _abi.EPI_STORE, "bias_relu": _abi.EPI_BIAS_RELU}[epi]
    K.conv_window(_abi.CONV_FPROP, Xs, k2, d, Wt, ld, out, cs, epilogue=code, bias=bias)
    ref = torch.nn.functional.conv2d(X.permute(0, 3, 1, 2).double().cpu(), W.double().cpu(), stride=4)
    ref = ref.permute(0, 2, 3, 1).reshape(-1, d)
    if epi == "bias_relu":
        ref = (ref + bias.double().cpu()).clamp_min(0)
    torch.cuda.synchronize()
    o = out.cpu()
    assert torch.isnan(o[:, d:]).all()
    assert rel_err(o[:, :d], ref) < 2e-3


@pytest.mark.parametrize("b,d", [(1, 96), (6, 96), (3, 64), (2, 32), (20, 96)])
def test_conv_window_wgrad_bias_vs_torch(b, d):
    """Weight + bias gradient of the space-to-depth conv1 through the window
    wgrad kernel (M = (kx, ky*48 + ch) in 32-channel MN-major atoms over the
    overlapping-row view; s2d rows resident in a ring across output rows;
    b = 20: 7-8 output rows per CTA, the ring wraps and runs cross images), mapped back
    to OIHW, against torch's conv2d weight grad."""
    gen = torch.Generator().manual_seed(70 + b)
    X, W, Xs, k2, n2, cp = _s2d_conv1(b, gen, d=d)
    m = n2 - k2 + 1
    dY = torch.randn(b * m * m, d, generator=gen)
    ldw = K.round_up(k2 * k2 * cp + 16, 32)
    dWt = torch.full((d, ldw), float("nan"), device=DEV)
    K.conv_window(_abi.CONV_WGRAD_BIAS, Xs, k2, d, dY.to(DEV), d, dWt, ldw)
    dW = torch.empty(d, 3, 11, 11, device=DEV)
    db = torch.empty(d, device=DEV)
    K.conv_weight_s2d(dW, d, 3, 11, 4, cp, dWt, ldw, inverse=True, bias=db)
    Xd = X.permute(0, 3, 1, 2).double().cpu()
    Wd = W.double().cpu().requires_grad_(True)
    ref = torch.nn.functional.conv2d(Xd, Wd, stride=4)
    ref.backward(dY.reshape(b, m, m, d).permute(0, 3, 1, 2).double())
    torch.cuda.synchronize()
    assert rel_err(dW.cpu(), Wd.grad) < 2e-3
    assert rel_err(db.cpu(), dY.double().sum(0)) < 2e-3   # the bias row is a TF32 product too


@pytest.mark.parametrize("prec", ["tf32", "3xtf32"])
def test_conv_implicit_partial_channel_block(prec):
    """d_in = 48 (the window path's space-to-depth image): the generic implicit
    GEMM runs 64-wide per-tap channel blocks whose last 16 channels read as
    zeros (TMA out-of-bounds fill), fprop and wgrad + bias row, vs torch."""
    gen = torch.Generator().manual_seed(81)
    X, W, Xs, k2, n2, cp = _s2d_conv1(3, gen)
    d, m = 96, n2 - k2 + 1
    ld = K.round_up(k2 * k2 * 64 + 1, 32)
    Wt = torch.zeros(d, ld, device=DEV)
    K.conv_weight_s2d(W, d, 3, 11, 4, 64, Wt, ld)          # 64 weight columns per tap
    pc = {"tf32": _abi.PREC_TF32, "3xtf32": _abi.PREC_3XTF32}[prec]
    tol = 2e-3 if prec == "tf32" else 1e-5
    out = torch.empty(3 * m * m, d, device=DEV)
    K.conv_implicit(_abi.CONV_FPROP, Xs, cp, k2, 1, 0, d, Wt, ld, out, d, precision=pc)
    Xd = X.permute(0, 3, 1, 2).double().cpu()
    Wd = W.double().cpu().requires_grad_(True)
    ref = torch.nn.functional.conv2d(Xd, Wd, stride=4)
    torch.cuda.synchronize()
    assert rel_err(out.cpu(), ref.permute(0, 2, 3, 1).reshape(-1, d)) < tol
    dY = torch.randn(3 * m * m, d, generator=gen)
    ref.backward(dY.reshape(3, m, m, d).permute(0, 3, 1, 2).double())
    dWt = torch.full((d, ld), float("nan"), device=DEV)
    K.conv_implicit(_abi.CONV_WGRAD_BIAS, Xs, cp, k2, 1, 0, d, dY.to(DEV), d, dWt, ld, precision=pc)
    dW = torch.empty(d, 3, 11, 11, device=DEV)
    db = torch.empty(d, device=DEV)
    K.conv_weight_s2d(dW, d, 3, 11, 4, 64, dWt, ld, inverse=True, bias=db)
    torch.cuda.synchronize()
    assert rel_err(dW.cpu(), Wd.grad) < tol
    assert rel_err(db.cpu(), dY.double().sum(0)) < max(tol, 1e-5)
