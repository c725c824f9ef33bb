"""Device-level wrappers: torch CUDA tensors in, libomni.so kernels out.

PyTorch is only the allocator and the stream provider here; every op below
is one (or two) launches of a hand-written sm_100a kernel through the C-ABI.
Strides ("ld") are in elements, as in include/omni.h.
"""

from __future__ import annotations

import ctypes

import torch

from . import _abi
from ._abi import call, query


def _ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:   # a host pointer would be dereferenced by the kernel (HMM/UVA)
        raise ValueError(f"libomni kernels take CUDA tensors (got {t.device}, shape {tuple(t.shape)})")
    return t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _require_cuda(*ts: torch.Tensor) -> None:
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("libomni kernels take CUDA tensors")


def _fits(t: torch.Tensor, need: int, name: str) -> None:
    """The kernels address operands as (pointer, ld): the storage behind the
    pointer must hold the whole strided extent, or a launch reads/writes past
    the allocation."""
    have = t.untyped_storage().nbytes() // t.element_size() - t.storage_offset()
    if need > have:
        raise ValueError(f"operand {name}: extent of {need} elements, only {have} behind the pointer")


def round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


# ----------------------------------------------------------------- K1 ----
def lower_nchw(D: torch.Tensor, k: int, stride: int, pad: int, start: int, b_p: int,
               ld: int | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
    """Reference-order lowering of images [start, start+b_p) of NCHW ``D`` (tensors.py:164-181)."""
    _require_cuda(D)
    b, c, n, n2 = D.shape
    if n != n2:
        raise ValueError("lower expects square images")
    m = (n + 2 * pad - k) // stride + 1
    K = c * k * k
    ld = K if ld is None else ld
    if out is None:
        out = torch.empty((b_p * m * m, ld), dtype=D.dtype, device=D.device)
    D = D.contiguous()
    name = "omni_lower_nchw_f64" if D.dtype == torch.float64 else "omni_lower_nchw_f32"
    call(name, _ptr(D), b, c, n, k, stride, pad, start, b_p, _ptr(out), ld, _stream())
    return out


def lower_nhwc(X: torch.Tensor, c: int, k: int, stride: int, pad: int, ld: int,
               out: torch.Tensor | None = None, ones_col: bool = False) -> torch.Tensor:
    """Tap-major lowering of NHWC activations (pixel stride X.shape[3]); ones_col
    writes 1.0 into column c*k*k (bias folded into the GEMM)."""
    _require_cuda(X)
    b, n, _, cs = X.shape
    m = (n + 2 * pad - k) // stride + 1
    if out is None:
        out = torch.empty((b * m * m, ld), dtype=torch.float32, device=X.device)
    call("omni_lower_nhwc_f32", _ptr(X), b, n, c, cs, k, stride, pad, int(ones_col), _ptr(out), ld,
         _stream())
    return out


def lift_nchw(Rhat: torch.Tensor, b: int, m: int, d_out: int) -> torch.Tensor:
    """(b*m^2, d_out) GEMM output -> NCHW tensor (tensors.py:213-219)."""
    _require_cuda(Rhat)
    out = torch.empty((b, d_out, m, m), dtype=Rhat.dtype, device=Rhat.device)
    name = "omni_lift_nchw_f64" if Rhat.dtype == torch.float64 else "omni_lift_nchw_f32"
    call(name, _ptr(Rhat), Rhat.stride(0), b, m, d_out, _ptr(out), _stream())
    return out


def col2im_nhwc(dDhat: torch.Tensor, ld: int, b: int, n: int, c: int, cs: int, k: int,
                stride: int, pad: int, dX: torch.Tensor,
                relu_mask: torch.Tensor | None = None) -> torch.Tensor:
    call("omni_col2im_nhwc_f32", _ptr(dDhat), ld, b, n, c, cs, k, stride, pad, _ptr(relu_mask),
         _ptr(dX), _stream())
    return dX


# ----------------------------------------------------------------- K2 ----
_ws_cache: dict[int, torch.Tensor] = {}


def gemm_workspace_bytes(precision: int, M: int, N: int, K: int, a_mn: bool, b_mn: bool) -> int:
    return int(query("omni_gemm_plan", precision, M, N, K, int(a_mn), int(b_mn), None, None))


def gemm_plan(precision: int, M: int, N: int, K: int) -> tuple[int, int]:
    import ctypes

    s = ctypes.c_int(0)
    bn = ctypes.c_int(0)
    query("omni_gemm_plan", precision, M, N, K, 0, 0, ctypes.byref(s), ctypes.byref(bn))
    return s.value, bn.value


def _workspace(nbytes: int, device: torch.device) -> torch.Tensor | None:
    if nbytes <= 0:
        return None
    key = device.index if device.index is not None else torch.cuda.current_device()
    ws = _ws_cache.get(key)
    if ws is None or ws.numel() * 4 < nbytes:
        ws = torch.empty((nbytes + 3) // 4, dtype=torch.float32, device=device)
        _ws_cache[key] = ws
    return ws


def _check_workspace(need: int, workspace: torch.Tensor | None, device) -> torch.Tensor | None:
    """A caller-owned workspace must be big enough (engines size theirs per
    launch; sharing a fallback buffer across streams or CUDA graphs would
    race).  Without one, standalone calls use a per-device cache."""
    if need <= 0:
        return workspace
    if workspace is not None:
        if workspace.numel() * 4 < need:
            raise RuntimeError(f"split-K workspace of {need} bytes needed, "
                               f"{workspace.numel() * 4} given")
        return workspace
    if torch.cuda.is_current_stream_capturing():
        raise RuntimeError("split-K GEMM inside CUDA graph capture needs an explicit workspace")
    return _workspace(need, device)


def gemm(M: int, N: int, K: int, A: torch.Tensor, lda: int, a_mn: bool, B: torch.Tensor,
         ldb: int, b_mn: bool, C: torch.Tensor, ldc: int, *, precision: int = _abi.PREC_TF32,
         epilogue: int = _abi.EPI_STORE, bias: torch.Tensor | None = None,
         aux: torch.Tensor | None = None, ld_aux: int = 0,
         workspace: torch.Tensor | None = None) -> torch.Tensor:
    """C[i,j] (op)= sum_r A(i,r) B(j,r) on tcgen05 (see include/omni.h for the operand maps)."""
    _require_cuda(A, B, C)
    if M > 0 and N > 0 and K > 0:
        _fits(A, (K - 1) * lda + M if a_mn else (M - 1) * lda + K, "A")
        _fits(B, (K - 1) * ldb + N if b_mn else (N - 1) * ldb + K, "B")
        _fits(C, (M - 1) * ldc + N, "C")
        if aux is not None:
            _fits(aux, (M - 1) * ld_aux + N, "aux")
        if bias is not None:
            _fits(bias, N, "bias")
    need = gemm_workspace_bytes(precision, M, N, K, a_mn, b_mn)
    workspace = _check_workspace(need, workspace, C.device)
    call("omni_gemm_f32", precision, M, N, K, _ptr(A), lda, int(a_mn), _ptr(B), ldb, int(b_mn),
         _ptr(C), ldc, epilogue, _ptr(bias), _ptr(aux), ld_aux, _ptr(workspace),
         0 if workspace is None else workspace.numel() * 4, _stream())
    return C


def matmul(A: torch.Tensor, B: torch.Tensor, precision: int = _abi.PREC_3XTF32) -> torch.Tensor:
    """Plain (M x K) @ (K x N) product of dense fp32 CUDA matrices on tcgen05."""
    M, K = A.shape
    K2, N = B.shape
    if K != K2:
        raise ValueError(f"inner dimensions disagree: {tuple(A.shape)} x {tuple(B.shape)}")
    lda = round_up(K, 4)
    if A.stride(0) != lda or A.stride(1) != 1 or A.data_ptr() % 16:
        Ap = torch.zeros((M, lda), dtype=torch.float32, device=A.device)
        Ap[:, :K] = A
    else:
        Ap = A
    ldb = round_up(N, 4)
    if B.stride(0) != ldb or B.stride(1) != 1 or B.data_ptr() % 16:
        Bp = torch.zeros((K, ldb), dtype=torch.float32, device=B.device)
        Bp[:, :N] = B
    else:
        Bp = B
    C = torch.empty((M, N), dtype=torch.float32, device=A.device)
    # A is K-major; B (K x N row-major) is MN-major for the B(j, r) operand.
    return gemm(M, N, K, Ap, lda, False, Bp, ldb, True, C, N, precision=precision)


def conv_implicit_workspace_bytes(precision: int, op: int, b: int, n: int, c: int, k: int,
                                  stride: int, pad: int, d_out: int) -> int:
    return int(query("omni_conv_implicit_plan", precision, op, b, n, c, k, stride, pad, d_out))


def conv_implicit(op: int, X: torch.Tensor, c: int, k: int, stride: int, pad: int, d_out: int,
                  G: torch.Tensor, ldg: int, Y: torch.Tensor, ldy: int, *,
                  precision: int = _abi.PREC_TF32, epilogue: int = _abi.EPI_STORE,
                  bias: torch.Tensor | None = None, aux: torch.Tensor | None = None,
                  ld_aux: int = 0, workspace: torch.Tensor | None = None) -> torch.Tensor:
    """Implicit-GEMM conv (TMA im2col operands) -- see include/omni.h.  X is NHWC
    (b, n, n, cs); op = _abi.CONV_FPROP, _abi.CONV_WGRAD or _abi.CONV_WGRAD_BIAS (the
    bias gradient lands in column k*k*c of Y)."""
    _require_cuda(X, G, Y)
    b, n, _, cs = X.shape
    m = (n + 2 * pad - k) // stride + 1
    pixels, taps = b * m * m, k * k * round_up(c, 32)   # cp = round_up(c, 32) per tap
    _fits(X, (b * n * n - 1) * cs + c, "X")
    if op == _abi.CONV_FPROP:   # G: d_out x ldg (tap-major weights), Y: pixels x ldy
        _fits(G, (d_out - 1) * ldg + taps, "G")
        _fits(Y, (pixels - 1) * ldy + d_out, "Y")
        if aux is not None:
            _fits(aux, (pixels - 1) * ld_aux + d_out, "aux")
    else:                       # G: dY, pixels x ldg; Y: dW (+ bias column), d_out x ldy
        _fits(G, (pixels - 1) * ldg + d_out, "G")
        _fits(Y, (d_out - 1) * ldy + taps + (op == _abi.CONV_WGRAD_BIAS), "Y")
    if bias is not None:
        _fits(bias, d_out, "bias")
    need = conv_implicit_workspace_bytes(precision, op, b, n, c, k, stride, pad, d_out)
    workspace = _check_workspace(need, workspace, Y.device)
    call("omni_conv_implicit_f32", precision, op, _ptr(X), b, n, c, cs, k, stride, pad, d_out,
         _ptr(G), ldg, _ptr(Y), ldy, epilogue, _ptr(bias), _ptr(aux), ld_aux, _ptr(workspace),
         0 if workspace is None else workspace.numel() * 4, _stream())
    return Y


def conv_window_plan(op: int, b: int, n2: int, cp: int, k2: int, d_out: int) -> int:
    """Workspace bytes of the space-to-depth window conv, or -1 if it does not apply."""
    return int(_abi.query("omni_conv_window_plan", op, b, n2, cp, k2, d_out))


def conv_window(op: int, Xs: torch.Tensor, k2: int, d_out: int, G: torch.Tensor, ldg: int,
                Y: torch.Tensor, ldy: int, *, epilogue: int = _abi.EPI_STORE,
                bias: torch.Tensor | None = None, workspace: torch.Tensor | None = None) -> torch.Tensor:
    """Window implicit GEMM of a space-to-depth first layer (see include/omni.h):
    Xs (b, n2, n2, 48); op = _abi.CONV_FPROP (G weights, Y NHWC output rows) or
    _abi.CONV_WGRAD_BIAS (G = dZ rows, Y = staged dW with the bias in column k2*k2*48)."""
    _require_cuda(Xs, G, Y)
    b, n2, _, cp = Xs.shape
    m = n2 - k2 + 1
    pixels, taps = b * m * m, k2 * k2 * cp
    if op == _abi.CONV_FPROP:
        _fits(G, (d_out - 1) * ldg + taps, "G")
        _fits(Y, (pixels - 1) * ldy + d_out, "Y")
    else:
        _fits(G, (pixels - 1) * ldg + d_out, "G")
        _fits(Y, (d_out - 1) * ldy + taps + 4, "Y")
        # the overlapping-row view of Xs reads 16 floats past its last pixel
        slack = Xs.untyped_storage().nbytes() // 4 - Xs.storage_offset() - Xs.numel()
        if not Xs.is_contiguous() or slack < 16:
            raise ValueError("conv_window wgrad: Xs must be contiguous with >= 16 readable floats after it")
    if bias is not None:
        _fits(bias, d_out, "bias")
    need = conv_window_plan(op, b, n2, cp, k2, d_out)
    if need < 0:
        raise ValueError(f"conv_window: geometry not covered (b={b} n2={n2} cp={cp} k2={k2} d_out={d_out})")
    workspace = _check_workspace(need, workspace, Y.device)
    call("omni_conv_window_f32", op, _ptr(Xs), b, n2, cp, k2, d_out, _ptr(G), ldg, _ptr(Y), ldy, epilogue,
         _ptr(bias), _ptr(workspace), 0 if workspace is None else workspace.numel() * 4, _stream())
    return Y


def conv_weight_flip(W: torch.Tensor, o: int, c: int, k: int, Wf: torch.Tensor, ld: int) -> None:
    call("omni_conv_weight_flip_f32", _ptr(W), o, c, k, _ptr(Wf), ld, _stream())


# ----------------------------------------------------------------- K3 ----
def pool_out_size(n: int, k: int, stride: int, pad: int, ceil_mode: bool) -> int:
    v = query("omni_pool_out_size", n, k, stride, pad, int(ceil_mode))
    if v < 1:
        raise ValueError(f"invalid pooling geometry n={n} k={k} s={stride} p={pad}")
    return int(v)


def pool_fwd(mode: int, X: torch.Tensor, c: int, k: int, stride: int, pad: int, ceil_mode: bool,
             Y: torch.Tensor, argmax: torch.Tensor | None) -> None:
    b, h, w, cs_in = X.shape
    call("omni_pool_fwd_nhwc_f32", mode, _ptr(X), b, h, w, c, cs_in, k, stride, pad,
         int(ceil_mode), _ptr(Y), Y.shape[3], _ptr(argmax), _stream())


def pool_bwd(mode: int, dY: torch.Tensor, X_shape, c: int, k: int, stride: int, pad: int,
             ceil_mode: bool, argmax: torch.Tensor | None, X: torch.Tensor | None,
             relu_mask: int, dX: torch.Tensor) -> None:
    """relu_mask: 0 none, 1 mask by (X > 0) with X the pool input, 2 (max pool)
    mask by (Y > 0) with X the pooled output -- see include/omni.h."""
    b, h, w, cs_in = X_shape
    call("omni_pool_bwd_nhwc_f32", mode, _ptr(dY), b, h, w, c, cs_in, k, stride, pad,
         int(ceil_mode), dY.shape[3], _ptr(argmax), _ptr(X), int(relu_mask), _ptr(dX), _stream())


# ----------------------------------------------------------------- K4 ----
def softmax_xent(logits: torch.Tensor, ld: int, labels: torch.Tensor, b: int, C: int,
                 loss: torch.Tensor, dlogits: torch.Tensor | None, ldd: int, scale: float) -> None:
    call("omni_softmax_xent_f32", _ptr(logits), ld, _ptr(labels), b, C, _ptr(loss),
         _ptr(dlogits), ldd, scale, _stream())


# ---------------------------------------------------------------- misc ---
def relu_fwd(X: torch.Tensor, Y: torch.Tensor) -> None:
    call("omni_relu_fwd_f32", _ptr(X), _ptr(Y), X.numel(), _stream())


def relu_bwd(dY: torch.Tensor, Y: torch.Tensor, dX: torch.Tensor) -> None:
    call("omni_relu_bwd_f32", _ptr(dY), _ptr(Y), _ptr(dX), dY.numel(), _stream())


def bias_grad_ws_elems(M: int, N: int) -> int:
    return int(query("omni_bias_grad_ws_elems", M, N))


def bias_grad(dY: torch.Tensor, ld: int, M: int, N: int, db: torch.Tensor,
              ws: torch.Tensor) -> None:
    call("omni_bias_grad_f32", _ptr(dY), ld, M, N, _ptr(db), _ptr(ws), _stream())


def sgd_momentum(W: torch.Tensor, V: torch.Tensor, g: torch.Tensor, w_read: torch.Tensor,
                 eta: float, mu: float, lam: float) -> None:
    call("omni_sgd_momentum_f32", _ptr(W), _ptr(V), _ptr(g), _ptr(w_read), eta, mu, lam,
         W.numel(), _stream())


def sgd_momentum_f64(W: torch.Tensor, V: torch.Tensor, g: torch.Tensor, w_read: torch.Tensor,
                     eta: float, mu: float, lam: float) -> None:
    """float64 K8 (bit-identical to the reference's NumPy update)."""
    for t in (W, V, g, w_read):
        if t.dtype != torch.float64:
            raise ValueError("sgd_momentum_f64 takes float64 tensors")
    call("omni_sgd_momentum_f64", _ptr(W), _ptr(V), _ptr(g), _ptr(w_read), eta, mu, lam,
         W.numel(), _stream())


def group_updates(rows: torch.Tensor, members: list, W: torch.Tensor, V: torch.Tensor,
                  snaps: list, eta: float, mu: float, lam: float) -> None:
    """The g ordered updates of a compute-group round on one shard (one
    kernel): rows is (nrows, >= n) with unit inner stride, row m = rank m's
    gradient shard; members[i] lists group i's rows in summation order;
    snaps[i] is group i's snapshot (the regulariser's w_read, overwritten
    with W after update i)."""
    n = W.numel()
    if rows.dim() != 2 or rows.stride(1) != 1 or rows.shape[1] < n:
        raise ValueError("group_updates: rows must be (nrows, >= n) with unit inner stride")
    g, k = len(members), len(members[0])
    if len(snaps) != g or any(len(m) != k for m in members):
        raise ValueError("group_updates: one snapshot and k members per group")
    if any(t.numel() != n or not t.is_contiguous() for t in (V, *snaps)) or not W.is_contiguous():
        raise ValueError("group_updates: W, V and the snapshots must be contiguous shards of equal length")
    mem = (ctypes.c_int * (g * k))(*[m for ms in members for m in ms])
    sp = (ctypes.c_void_p * g)(*[t.data_ptr() for t in snaps])
    call("omni_group_updates_f32", _ptr(rows), rows.shape[0], rows.stride(0), mem, g, k, _ptr(W),
         _ptr(V), sp, n, eta, mu, lam, _stream())


def gather_rows(src: torch.Tensor, idx: torch.Tensor, dst: torch.Tensor) -> None:
    row = src[0].numel()
    call("omni_gather_rows_f32", _ptr(src), row, _ptr(idx), idx.numel(), _ptr(dst), _stream())


def gather_i32(src: torch.Tensor, idx: torch.Tensor, dst: torch.Tensor) -> None:
    call("omni_gather_i32", _ptr(src), _ptr(idx), idx.numel(), _ptr(dst), _stream())


def conv_weight_to_tap(W: torch.Tensor, o: int, c: int, k: int, Wt: torch.Tensor, ld: int,
                       inverse: bool = False, bias: torch.Tensor | None = None) -> None:
    call("omni_conv_weight_to_tap_f32", _ptr(W), o, c, k, _ptr(Wt), ld, int(inverse), _ptr(bias),
         _stream())


def space_to_depth(X: torch.Tensor, c: int, s: int, Y: torch.Tensor) -> None:
    """NHWC X (b, n, n, cs) -> Y (b, n2, n2, cp) (see include/omni.h)."""
    b, n, _, cs = X.shape
    call("omni_space_to_depth_f32", _ptr(X), b, n, c, cs, s, _ptr(Y), Y.shape[1], Y.shape[3],
         _stream())


def space_to_depth_gather(data: torch.Tensor, idx: torch.Tensor, c: int, s: int,
                          Y: torch.Tensor) -> None:
    """Y[i] = space_to_depth(data[idx[i]]): batch gather fused into the transform."""
    _require_cuda(data, idx, Y)
    if idx.dtype != torch.int64:
        raise ValueError("idx must be int64")
    _, n, _, cs = data.shape
    b = idx.numel()
    _fits(Y, b * Y.shape[1] * Y.shape[2] * Y.shape[3], "Y")
    call("omni_space_to_depth_gather_f32", _ptr(data), _ptr(idx), b, n, c, cs, s, _ptr(Y),
         Y.shape[1], Y.shape[3], _stream())


def conv_weight_s2d(W: torch.Tensor, o: int, c: int, k: int, s: int, cp: int, Wt: torch.Tensor,
                    ld: int, inverse: bool = False, bias: torch.Tensor | None = None) -> None:
    call("omni_conv_weight_s2d_f32", _ptr(W), o, c, k, s, cp, _ptr(Wt), ld, int(inverse),
         _ptr(bias), _stream())


def transpose(src: torch.Tensor, lds: int, src_bstride: int, rows: int, cols: int,
              dst: torch.Tensor, ldd: int, dst_bstride: int, batch: int = 1) -> None:
    call("omni_transpose_f32", _ptr(src), lds, src_bstride, rows, cols, _ptr(dst), ldd,
         dst_bstride, batch, _stream())


def fill(X: torch.Tensor, value: float) -> None:
    call("omni_fill_f32", _ptr(X), float(value), X.numel(), _stream())
