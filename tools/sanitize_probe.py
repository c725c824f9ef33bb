"""One small launch of every libomni kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python tools/sanitize_probe.py

GEMM: single CTA, CTA pair, 3xTF32 (converter warps), split-K + reduce, TMA
store and direct epilogues; implicit conv fprop / wgrad(+bias row) / dgrad
(flipped weights), transposed fprop, partial channel block; the conv1 window
kernels; lowering / col2im / lift; pooling; softmax-CE; bias gradient; SGD
(fp32 and fp64); gathers and space-to-depth.  Exits 0 after a final
synchronize (an error raises).
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1606_04487_b200 import _abi, kernels as K  # noqa: E402

DEV = "cuda"


def main():
    g = torch.Generator(device=DEV).manual_seed(0)
    r = lambda *s: torch.randn(*s, device=DEV, generator=g)  # noqa: E731
    # ---- GEMM variants
    for prec in (_abi.PREC_TF32, _abi.PREC_3XTF32):
        for (M, N, Kd) in ((300, 96, 200), (64, 40, 5000), (257, 256, 64)):
            A, B = r(M, K.round_up(Kd, 4)), r(N, K.round_up(Kd, 4))
            C = torch.empty(M, K.round_up(N, 4), device=DEV)
            K.gemm(M, N, Kd, A, A.shape[1], False, B, B.shape[1], False, C, C.shape[1], precision=prec)
            bias = r(N)
            K.gemm(M, N, Kd, A, A.shape[1], False, B, B.shape[1], False, C, C.shape[1], precision=prec,
                   epilogue=_abi.EPI_BIAS_RELU, bias=bias)
    # ---- implicit conv (b=2, 13x13x64 -> 32, k3 p1) fprop / wgrad+bias / dgrad
    b, n, c, k, p, d = 2, 13, 64, 3, 1, 32
    X = r(b, n, n, c)
    ld = K.round_up(k * k * c + 1, 32)
    Wt = r(d, ld)
    Y = torch.empty(b * n * n, d, device=DEV)
    for prec in (_abi.PREC_TF32, _abi.PREC_3XTF32):
        K.conv_implicit(_abi.CONV_FPROP, X, c, k, 1, p, d, Wt, ld, Y, d, precision=prec,
                        epilogue=_abi.EPI_BIAS_RELU, bias=r(d))
        dW = torch.empty(d, ld, device=DEV)
        K.conv_implicit(_abi.CONV_WGRAD_BIAS, X, c, k, 1, p, d, r(b * n * n, d), d, dW, ld, precision=prec)
        Wf = r(c, K.round_up(d * k * k, 32))
        dX = torch.empty(b * n * n, c, device=DEV)
        K.conv_implicit(_abi.CONV_FPROP, r(b, n, n, d), d, k, 1, k - 1 - p, c, Wf, Wf.shape[1], dX, c,
                        precision=prec, epilogue=_abi.EPI_MASK_AUX, aux=X.view(-1, c), ld_aux=c)
    # ---- space-to-depth first layer: window fprop, generic wgrad over 48 channels
    b, n = 2, 227
    X1 = r(b, n, n, 3)
    Xs = torch.zeros(b, 57, 57, 48, device=DEV)
    K.space_to_depth(X1, 3, 4, Xs)
    idx = torch.tensor([1, 0], device=DEV, dtype=torch.int64)
    K.space_to_depth_gather(X1, idx, 3, 4, Xs)
    W1 = r(96, 3, 11, 11)
    Wt1 = torch.zeros(96, 448, device=DEV)
    K.conv_weight_s2d(W1, 96, 3, 11, 4, 48, Wt1, 448)
    Y1 = torch.empty(b * 55 * 55, 96, device=DEV)
    K.conv_window(_abi.CONV_FPROP, Xs, 3, 96, Wt1, 448, Y1, 96, epilogue=_abi.EPI_BIAS_RELU, bias=r(96))
    dW1 = torch.empty(96, 608, device=DEV)
    K.conv_implicit(_abi.CONV_WGRAD_BIAS, Xs, 48, 3, 1, 0, 96, r(b * 55 * 55, 96), 96, dW1, 608)
    dWw = torch.empty(96, 448, device=DEV)
    K.conv_window(_abi.CONV_WGRAD_BIAS, Xs, 3, 96, r(b * 55 * 55, 96), 96, dWw, 448)
    # ---- lowering / col2im / lift (explicit layers)
    Xl = r(2, 12, 12, 20)
    ldl = K.round_up(20 * 25 + 1, 32)
    Dh = torch.empty(2 * 8 * 8, ldl, device=DEV)
    K.lower_nhwc(Xl, 20, 5, 1, 0, ldl, out=Dh, ones_col=True)
    dXl = torch.empty(2, 12, 12, 20, device=DEV)
    K.col2im_nhwc(Dh, ldl, 2, 12, 20, 20, 5, 1, 0, dXl, None)
    # ---- pooling, softmax, bias grad, sgd, gathers
    Xp = r(4, 27, 27, 96)
    o = K.pool_out_size(27, 3, 2, 0, True)
    Yp = torch.empty(4, o, o, 96, device=DEV)
    arg = torch.empty(4 * o * o * 96, dtype=torch.int32, device=DEV)
    K.pool_fwd(0, Xp, 96, 3, 2, 0, True, Yp, arg)
    dXp = torch.empty_like(Xp)
    K.pool_bwd(0, r(4, o, o, 96), (4, 27, 27, 96), 96, 3, 2, 0, True, arg, Yp, 2, dXp)
    K.pool_fwd(1, Xp, 96, 3, 2, 0, True, Yp, None)
    logits = r(8, 1000)
    lab = torch.randint(0, 1000, (8,), device=DEV, dtype=torch.int32)
    loss = torch.empty(1, device=DEV)
    dl = torch.empty_like(logits)
    K.softmax_xent(logits, 1000, lab, 8, 1000, loss, dl, 1000, 1.0 / 8)
    db = torch.empty(1000, device=DEV)
    K.bias_grad(dl, 1000, 8, 1000, db, torch.empty(K.bias_grad_ws_elems(8, 1000), device=DEV))
    W, V, G = r(10001), r(10001), r(10001)
    K.sgd_momentum(W, V, G, W, 0.01, 0.9, 5e-4)
    Wd, Vd, Gd = W.double(), V.double(), G.double()
    K.sgd_momentum_f64(Wd, Vd, Gd, Wd, 0.01, 0.9, 5e-4)
    src = r(16, 33)
    dst = torch.empty(4, 33, device=DEV)
    K.gather_rows(src, torch.tensor([3, 1, 15, 0], device=DEV), dst)
    torch.cuda.synchronize()
    print("sanitize probe: all kernel families launched and synchronized")


if __name__ == "__main__":
    main()
