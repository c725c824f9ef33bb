"""Time (or profile under ncu) one implicit-GEMM conv launch.

    python tools/conv_probe.py op b n c k s p d_out [reps]      (op: fprop | wgrad)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1606_04487_b200 import _abi, kernels as K  # noqa: E402


def main():
    op = sys.argv[1]
    b, n, c, k, s, p, d = (int(v) for v in sys.argv[2:9])
    reps = int(sys.argv[9]) if len(sys.argv) > 9 else 10
    dev = torch.device("cuda")
    m = (n + 2 * p - k) // s + 1
    X = torch.randn(b, n, n, c, device=dev)
    ld = K.round_up(c * k * k, 32)
    if op == "fprop":
        G = torch.randn(d, ld, device=dev)
        Y = torch.empty(b * m * m, d, device=dev)
        args = (_abi.CONV_FPROP, X, c, k, s, p, d, G, ld, Y, d)
        flops = 2.0 * b * m * m * d * c * k * k
    else:
        G = torch.randn(b * m * m, d, device=dev)
        Y = torch.empty(d, ld, device=dev)
        args = (_abi.CONV_WGRAD, X, c, k, s, p, d, G, d, Y, ld)
        flops = 2.0 * b * m * m * d * c * k * k
    for _ in range(2):
        K.conv_implicit(*args)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        K.conv_implicit(*args)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{op} b={b} n={n} c={c} k={k} s={s} p={p} d={d}: {ms:.3f} ms {flops / ms / 1e9:.1f} TFLOP/s")


if __name__ == "__main__":
    main()
