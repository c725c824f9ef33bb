"""Time CaffeNet conv1 (b=256) through the window kernels (conv_window.cu,
cp = 48) and through the generic implicit GEMM (cp = 64), CUDA events.

    python tools/window_probe.py [--reps N] [--once]      (--once: one launch each, for ncu)
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1606_04487_b200 import _abi, kernels as K  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--once", action="store_true")
    ap.add_argument("--b", type=int, default=256)
    a = ap.parse_args()
    b, n, c, k, s, d = a.b, 227, 3, 11, 4, 96
    k2, n2, m = 3, 57, 55
    dev = "cuda"
    X = torch.randn(b, n, n, c, device=dev)
    W = torch.randn(d, c, k, k, device=dev) / (c * k * k) ** 0.5
    bias = torch.randn(d, device=dev)
    dY = torch.randn(b * m * m, d, device=dev)
    out = torch.empty(b * m * m, d, device=dev)
    res = {}
    for cp, kind in ((48, "window"), (64, "implicit")):
        Xs = torch.zeros(b * n2 * n2 * cp + 64, device=dev)[:b * n2 * n2 * cp].view(b, n2, n2, cp)
        K.space_to_depth(X, c, s, Xs)
        ld = K.round_up(k2 * k2 * cp, 32)
        Wt = torch.zeros(d, ld, device=dev)
        K.conv_weight_s2d(W, d, c, k, s, cp, Wt, ld)
        ldw = K.round_up(k2 * k2 * cp + 16, 32)
        dWt = torch.empty(d, ldw, device=dev)
        if kind == "window":
            ws = torch.empty(max(K.conv_window_plan(_abi.CONV_WGRAD_BIAS, b, n2, cp, k2, d), 16) // 4, device=dev)
            fprop = lambda: K.conv_window(_abi.CONV_FPROP, Xs, k2, d, Wt, ld, out, d,  # noqa: E731
                                          epilogue=_abi.EPI_BIAS_RELU, bias=bias)
            wgrad = lambda: K.conv_window(_abi.CONV_WGRAD_BIAS, Xs, k2, d, dY, d, dWt, ldw,  # noqa: E731
                                          workspace=ws)
        else:
            need = max(K.conv_implicit_workspace_bytes(_abi.PREC_TF32, op, b, n2, cp, k2, 1, 0, d)
                       for op in (_abi.CONV_FPROP, _abi.CONV_WGRAD_BIAS))
            ws = torch.empty(max(need, 16) // 4, device=dev)
            fprop = lambda: K.conv_implicit(_abi.CONV_FPROP, Xs, cp, k2, 1, 0, d, Wt, ld, out, d,  # noqa: E731
                                            epilogue=_abi.EPI_BIAS_RELU, bias=bias, workspace=ws)
            wgrad = lambda: K.conv_implicit(_abi.CONV_WGRAD_BIAS, Xs, cp, k2, 1, 0, d, dY, d, dWt, ldw,  # noqa: E731
                                            workspace=ws)
        for name, fn in (("fprop", fprop), ("wgrad", wgrad)):
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
            flops = 2.0 * b * m * m * d * c * k * k
            res[f"{kind}_{name}"] = {"ms": ms, "alg_tflops": flops / ms / 1e9}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
