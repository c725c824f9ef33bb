"""3xTF32 on CTA pairs (debug, OMNI_3X_PAIRS=1): normwise error of C = A B^T
against float64 per 128-row half of each 256-row pair tile, beside the
single-CTA 3xTF32 and TF32 errors (run once with and once without the env)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1606_04487_b200 import _abi, kernels as K  # noqa: E402


def main():
    torch.manual_seed(0)
    out = {"pairs_env": bool(os.environ.get("OMNI_3X_PAIRS"))}
    for (M, N, Kd) in ((512, 256, 512), (1024, 128, 256), (256, 256, 2048)):
        A = torch.randn(M, Kd, device="cuda")
        B = torch.randn(N, Kd, device="cuda")
        ref = A.double() @ B.double().T
        for name, prec in (("3xtf32", _abi.PREC_3XTF32), ("tf32", _abi.PREC_TF32)):
            C = torch.full((M, N), float("nan"), device="cuda")
            K.gemm(M, N, Kd, A, Kd, False, B, Kd, False, C, N, precision=prec)
            torch.cuda.synchronize()
            err = (C.double() - ref)
            halves = {}
            for h in (0, 1):
                rows = torch.cat([torch.arange(t * 256 + h * 128, t * 256 + h * 128 + 128)
                                  for t in range(M // 256)]) if M >= 256 else torch.arange(0)
                if rows.numel():
                    halves[f"rows_half{h}"] = float(err[rows].norm() / ref[rows].norm())
            out[f"{M}x{N}x{Kd}_{name}"] = {"rel": float(err.norm() / ref.norm()), **halves,
                                           "nan": bool(torch.isnan(C).any())}
    print(json.dumps(out, indent=1))


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def timing():
    """Time a large 3xTF32 GEMM (single CTAs vs pairs decided by the env)."""
    M = N = Kd = 4096
    A = torch.randn(M, Kd, device="cuda")
    B = torch.randn(N, Kd, device="cuda")
    C = torch.empty(M, N, device="cuda")
    for _ in range(2):
        K.gemm(M, N, Kd, A, Kd, False, B, Kd, False, C, N, precision=_abi.PREC_3XTF32)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        K.gemm(M, N, Kd, A, Kd, False, B, Kd, False, C, N, precision=_abi.PREC_3XTF32)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(json.dumps({"pairs_env": bool(os.environ.get("OMNI_3X_PAIRS")), "gemm_4096_3xtf32_ms": ms,
                      "tflops_effective": 2 * M * N * Kd / ms / 1e9}))


if len(sys.argv) > 1 and sys.argv[1] == "--timing":
    timing()
