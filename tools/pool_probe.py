"""Time the CaffeNet max-pool launches (b=256) alone with CUDA events: forward
(value + argmax) and the stride-2 backward (ReLU mask from the pooled output),
with achieved HBM GB/s from the bytes each must move.

    python tools/pool_probe.py [--reps N] [--once]     (--once: one launch each, for ncu)
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1606_04487_b200 import kernels as K  # noqa: E402

# (name, n, c): 3x3 / stride 2 max pools of CaffeNet (pool1, pool2, pool5)
LAYERS = [("pool1", 55, 96), ("pool2", 27, 256), ("pool5", 13, 256)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--once", action="store_true")
    ap.add_argument("--b", type=int, default=256)
    a = ap.parse_args()
    b, dev = a.b, "cuda"
    res = {}
    for name, n, c in LAYERS:
        m = K.pool_out_size(n, 3, 2, 0, False)
        X = torch.randn(b, n, n, c, device=dev)
        Y = torch.empty(b, m, m, c, device=dev)
        am = torch.empty(b, m, m, c, dtype=torch.int32, device=dev)
        dY = torch.randn(b, m, m, c, device=dev)
        dX = torch.empty(b, n, n, c, device=dev)
        fwd = lambda: K.pool_fwd(0, X, c, 3, 2, 0, False, Y, am)  # noqa: E731
        bwd = lambda: K.pool_bwd(0, dY, X.shape, c, 3, 2, 0, False, am, Y, 2, dX)  # noqa: E731
        # the engine's form: forward mode 2 (ReLU mask in the argmax sign bit), unmasked backward
        fwd2 = lambda: K.pool_fwd(2, X, c, 3, 2, 0, False, Y, am)  # noqa: E731
        bwd2 = lambda: K.pool_bwd(0, dY, X.shape, c, 3, 2, 0, False, am, None, 0, dX)  # noqa: E731
        xin, yout = 4 * b * n * n * c, 4 * b * m * m * c
        for kind, fn, nbytes in (("fwd", fwd, xin + 2 * yout), ("bwd", bwd, 3 * yout + xin),
                                 ("fwd_marked", fwd2, xin + 2 * yout), ("bwd_marked", bwd2, 2 * yout + xin)):
            fn()
            torch.cuda.synchronize()
            if a.once:
                continue
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            res[f"{name}_{kind}"] = {"us": ms * 1e3, "GBps": nbytes / ms / 1e6, "bytes": nbytes}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
