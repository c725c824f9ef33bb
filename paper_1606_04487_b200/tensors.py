"""Drop-in for omnisim.tensors: the conv operator API, computed on the B200.

Same names, argument meaning and ValueError messages as the reference
(tensors.py:31-261).  NumPy float64 in and out at this boundary; underneath:

* ``lower`` / ``lift``: K1 lowering and the lifting transpose, pure data
  movement in the caller's element type, so results are bit-identical to the
  reference for float64 inputs;
* ``gemm`` / ``conv_lowered``: one tcgen05 GEMM per call in 3xTF32 (default;
  ~fp32 accuracy, normwise relative error ~1e-6) or TF32 precision.  The
  reference computes in float64 with a fixed block order; this boundary
  states its tolerance instead of claiming bit-equality.

``b_p`` and ``workers`` keep their validation and meaning (b_p images per
GEMM, independent batch partitions); on the GPU neither changes the result.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _abi
from . import kernels as K

DEFAULT_PRECISION = "3xtf32"


def _dev():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1606_04487_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda")


@dataclass(frozen=True)
class ConvSpec:
    """Shape parameters of one convolution (tensors.py:31-59)."""

    n: int
    k: int
    d_in: int
    d_out: int
    stride: int = 1
    pad: int = 0

    def __post_init__(self) -> None:
        if min(self.n, self.k, self.d_in, self.d_out, self.stride) < 1:
            raise ValueError("n, k, d_in, d_out, stride must be positive")
        if self.pad < 0:
            raise ValueError("pad must be non-negative")
        if self.k > self.n + 2 * self.pad:
            raise ValueError(f"kernel {self.k} exceeds padded input {self.n + 2 * self.pad}")
        span = self.n + 2 * self.pad - self.k
        if span % self.stride != 0:
            raise ValueError(
                f"output size not integral: (n + 2*pad - k) = {span} "
                f"is not divisible by stride {self.stride}"
            )

    @property
    def m(self) -> int:
        return (self.n + 2 * self.pad - self.k) // self.stride + 1


@dataclass(frozen=True)
class Tensor4:
    """C-ordered (batch, channels, n1, n2) float64 container (tensors.py:62-112)."""

    values: np.ndarray

    def __post_init__(self) -> None:
        arr = np.ascontiguousarray(self.values, dtype=np.float64)
        if arr.ndim != 4:
            raise ValueError(f"expected 4 dims, got {arr.ndim}")
        if not np.all(np.isfinite(arr)):
            raise ValueError("tensor contains non-finite values")
        object.__setattr__(self, "values", arr)

    n1 = property(lambda self: self.values.shape[2])
    n2 = property(lambda self: self.values.shape[3])
    channels = property(lambda self: self.values.shape[1])
    batch = property(lambda self: self.values.shape[0])

    @property
    def dims(self) -> tuple[int, int, int, int]:
        return (self.n1, self.n2, self.channels, self.batch)

    @property
    def data(self) -> np.ndarray:
        return self.values.ravel()

    @classmethod
    def from_flat(cls, dims, data) -> "Tensor4":
        n1, n2, channels, batch = dims
        arr = np.asarray(data, dtype=np.float64)
        if arr.size != n1 * n2 * channels * batch:
            raise ValueError(
                f"data length {arr.size} != n1*n2*channels*batch = {n1 * n2 * channels * batch}"
            )
        return cls(arr.reshape(batch, channels, n1, n2))


@dataclass(frozen=True)
class LoweredMatrix:
    matrix: np.ndarray
    b_p: int

    rows = property(lambda self: self.matrix.shape[0])
    cols = property(lambda self: self.matrix.shape[1])

    @property
    def data(self) -> np.ndarray:
        return self.matrix.ravel()


def _check_conv_inputs(D: Tensor4, K_: Tensor4, spec: ConvSpec) -> None:
    if D.dims != (spec.n, spec.n, spec.d_in, D.batch):
        raise ValueError(f"data dims {D.dims} do not match spec (n={spec.n}, d_in={spec.d_in})")
    if K_.dims != (spec.k, spec.k, spec.d_in, K_.batch) or K_.batch != spec.d_out:
        raise ValueError(
            f"kernel dims {K_.dims} do not match spec (k={spec.k}, d_in={spec.d_in}, d_out={spec.d_out})"
        )


def lower(D: Tensor4, spec: ConvSpec, b_p: int, start: int = 0) -> LoweredMatrix:
    """Lower images [start, start+b_p) to (b_p*m^2, k^2*d_in) on the GPU (K1, float64, bit-exact)."""
    if not 1 <= b_p <= D.batch:
        raise ValueError(f"b_p={b_p} out of range [1, {D.batch}]")
    if not 0 <= start <= D.batch - b_p:
        raise ValueError(f"start={start} leaves fewer than b_p={b_p} images")
    Dd = torch.from_numpy(D.values).to(_dev())
    out = K.lower_nchw(Dd, spec.k, spec.stride, spec.pad, start, b_p)
    return LoweredMatrix(matrix=out.cpu().numpy(), b_p=b_p)


def lower_kernel(K_: Tensor4, spec: ConvSpec) -> np.ndarray:
    """(d_out, d_in, k, k) -> K-hat (d_in*k*k, d_out) (tensors.py:184-190).  A
    relayout of host memory only: on the device the OIHW weights are already
    K-hat^T, the GEMM's K-major operand, so the hot path never calls this."""
    if K_.dims != (spec.k, spec.k, spec.d_in, spec.d_out):
        raise ValueError(f"kernel dims {K_.dims} do not match spec")
    return np.ascontiguousarray(K_.values.reshape(spec.d_out, -1).T)


def _to_dev_padded(A: np.ndarray) -> tuple[torch.Tensor, int]:
    rows, cols = A.shape
    ld = K.round_up(cols, 4)
    t = torch.zeros((rows, ld), dtype=torch.float32, device=_dev())
    t[:, :cols] = torch.from_numpy(np.ascontiguousarray(A, dtype=np.float32))
    return t, ld


def gemm(A: np.ndarray, B: np.ndarray, precision: str = DEFAULT_PRECISION) -> np.ndarray:
    """R = A @ B on tcgen05 (K2).  float64 in/out; computed in 3xTF32 (default) or TF32."""
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    if A.ndim != 2 or B.ndim != 2:
        raise ValueError("gemm expects 2-D operands")
    if A.shape[1] != B.shape[0]:
        raise ValueError(f"inner dimensions disagree: {A.shape} x {B.shape}")
    M, Kd = A.shape
    N = B.shape[1]
    if M == 0 or N == 0:
        return np.zeros((M, N))
    if Kd == 0:
        return np.zeros((M, N))
    Ad, lda = _to_dev_padded(A)
    Bd, ldb = _to_dev_padded(B)   # (K x N) row-major: the MN-major B operand
    C = torch.empty((M, N), dtype=torch.float32, device=_dev())
    K.gemm(M, N, Kd, Ad, lda, False, Bd, ldb, True, C, N, precision=_abi.PRECISIONS[precision])
    return C.double().cpu().numpy()


def lift(Rhat: np.ndarray, spec: ConvSpec, b: int) -> Tensor4:
    """(b*m^2, d_out) -> NCHW Tensor4 on the GPU (float64, bit-exact) (tensors.py:213-219)."""
    Rhat = np.asarray(Rhat, dtype=np.float64)
    m = spec.m
    if Rhat.shape != (b * m * m, spec.d_out):
        raise ValueError(f"result shape {Rhat.shape} != ({b * m * m}, {spec.d_out})")
    out = K.lift_nchw(torch.from_numpy(np.ascontiguousarray(Rhat)).to(_dev()), b, m, spec.d_out)
    return Tensor4(out.cpu().numpy())


def conv_lowered_device(D: torch.Tensor, Kw: torch.Tensor, spec: ConvSpec, b_p: int,
                        precision: str = DEFAULT_PRECISION) -> torch.Tensor:
    """Device form of conv_lowered: D (b, d_in, n, n) fp32 NCHW, Kw (d_out, d_in, k, k)
    fp32 -> R (b, d_out, m, m) fp32.  b_p images share one GEMM."""
    b = D.shape[0]
    m = spec.m
    Kc = spec.d_in * spec.k * spec.k
    ld = K.round_up(Kc, 4)
    Wk = torch.zeros((spec.d_out, ld), dtype=torch.float32, device=D.device)
    Wk[:, :Kc] = Kw.reshape(spec.d_out, Kc)          # OIHW rows are K-hat^T (K-major B)
    Rhat = torch.empty((b * m * m, spec.d_out), dtype=torch.float32, device=D.device)
    Dhat = torch.empty((b_p * m * m, ld), dtype=torch.float32, device=D.device)
    for c0 in range(0, b, b_p):
        size = min(b_p, b - c0)
        K.lower_nchw(D, spec.k, spec.stride, spec.pad, c0, size, ld=ld, out=Dhat)
        rows = size * m * m
        K.gemm(rows, spec.d_out, Kc, Dhat, ld, False, Wk, ld, False, Rhat[c0 * m * m:], spec.d_out,
               precision=_abi.PRECISIONS[precision])
    return K.lift_nchw(Rhat, b, m, spec.d_out)


def conv_lowered(D: Tensor4, K_: Tensor4, spec: ConvSpec, b_p: int = 1, workers: int = 1,
                 precision: str = DEFAULT_PRECISION) -> Tensor4:
    """Convolution via lowering + one tcgen05 GEMM per b_p images + lifting (tensors.py:222-256)."""
    _check_conv_inputs(D, K_, spec)
    if not 1 <= b_p <= D.batch:
        raise ValueError(f"b_p={b_p} out of range [1, {D.batch}]")
    if workers < 1:
        raise ValueError("workers must be >= 1")
    dev = _dev()
    Dd = torch.from_numpy(D.values).to(device=dev, dtype=torch.float32)
    Kd = torch.from_numpy(K_.values).to(device=dev, dtype=torch.float32)
    # `workers` partitions the batch into independent GEMM streams on the CPU
    # reference; on the GPU the grid already spans all SMs, so partitions are
    # processed back to back with identical results.
    R = conv_lowered_device(Dd, Kd, spec, b_p, precision)
    return Tensor4(R.double().cpu().numpy())


def conv_direct(D: Tensor4, K_: Tensor4, spec: ConvSpec) -> Tensor4:
    """The reference's oracle route (tensors.py:144-161).  On the B200 there is
    one convolution engine, so this is conv_lowered with one GEMM per batch."""
    _check_conv_inputs(D, K_, spec)
    return conv_lowered(D, K_, spec, b_p=D.batch)


def blowup_ratio(spec: ConvSpec) -> float:
    """Replication factor of lowering: lowered elements / original elements."""
    return (spec.m ** 2 * spec.k ** 2) / spec.n ** 2
