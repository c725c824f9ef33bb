"""Time (or profile under ncu) one libomni GEMM shape standalone.

    python tools/gemm_probe.py M N K a_mn b_mn [precision] [reps]

Prints the CUDA-event time per launch and TFLOP/s.  Used for per-shape
roofline work and `ncu -k regex:gemm_tf32` captures.
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1606_04487_b200 import _abi, kernels as K  # noqa: E402


def main():
    M, N, Kd, a_mn, b_mn = (int(v) for v in sys.argv[1:6])
    prec = sys.argv[6] if len(sys.argv) > 6 else "tf32"
    reps = int(sys.argv[7]) if len(sys.argv) > 7 else 10
    dev = torch.device("cuda")
    lda = K.round_up(M if a_mn else Kd, 4)
    ldb = K.round_up(N if b_mn else Kd, 4)
    A = torch.randn((Kd if a_mn else M, lda), device=dev)
    B = torch.randn((Kd if b_mn else N, ldb), device=dev)
    ldc = K.round_up(N, 4)
    C = torch.empty((M, ldc), device=dev)
    p = _abi.PRECISIONS[prec]
    for _ in range(2):
        K.gemm(M, N, Kd, A, lda, bool(a_mn), B, ldb, bool(b_mn), C, ldc, precision=p)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        K.gemm(M, N, Kd, A, lda, bool(a_mn), B, ldb, bool(b_mn), C, ldc, precision=p)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    s, bn = K.gemm_plan(p, M, N, Kd)
    print(f"M={M} N={N} K={Kd} a_mn={a_mn} b_mn={b_mn} {prec} bn={bn} splits={s}: "
          f"{ms:.3f} ms  {2.0 * M * N * Kd / ms / 1e9:.1f} TFLOP/s")


if __name__ == "__main__":
    main()
