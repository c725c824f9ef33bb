"""Time the fused gather + space-to-depth of CaffeNet's input (b=256, 227x227x3
-> 57x57x48) alone with CUDA events; GB/s from the bytes it must move.

    python tools/s2d_probe.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1606_04487_b200 import kernels as K  # noqa: E402


def main():
    b, n, c, s = 256, 227, 3, 4
    X = torch.randn(b, n, n, c, device="cuda")
    idx = torch.randperm(b, device="cuda")
    Y = torch.empty(b, 57, 57, 48, device="cuda")
    K.space_to_depth_gather(X, idx, c, s, Y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        K.space_to_depth_gather(X, idx, c, s, Y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    nb = 4 * b * n * n * c + 4 * b * 57 * 57 * 48
    print(json.dumps({"us": ms * 1e3, "GBps": nb / ms / 1e6}))


if __name__ == "__main__":
    main()
