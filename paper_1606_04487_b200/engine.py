"""GpuNet: one NetSpec compiled into a fixed sequence of sm_100a launches.

This is the device-resident training step behind ``CNNProblem.grad`` and the
g-group runtime: the reference's problems.py:206-269 cascade (forward through
lowering + one GEMM per layer, softmax-CE, hand-written backward) and
sgd.py:92-101 update, for any NetSpec.

Layout in HBM (all fp32):
  * activations NHWC, pixel stride cs = round_up(c, 4) (16-byte rows for TMA
    and float4 kernels); FC activations (b, round_up(f, 4));
  * lowered matrices Dhat (b*m^2, round_up(c*k*k + bias, 32)) in tap-major
    column order (kx*k + ky)*c + ch (128-byte row pitch), kept from forward for
    the weight gradient;
  * conv weights staged each step from the flat OIHW vector into tap-major
    rows (the GEMM's K-major B operand); FC weights staged transposed
    (out, in) so the forward product is K-major x K-major;
  * the flat parameter / gradient vectors use the reference's packing
    (problems.py:201-204 generalised in nets.py).

Fusion: the conv bias rides in the GEMM itself (a ones column in Dhat and
the bias in the matching column of the staged weights, so the weight-gradient
GEMM also yields the bias gradient); ReLU in the GEMM epilogue; the ReLU mask
of the backward pass is applied by whichever kernel produces the gradient
(pool backward, col2im, FC dgrad epilogue).  Per-step launches are static, so the whole step can be captured in a
CUDA graph (``capture``).
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import torch

from . import _abi
from . import kernels as K
from .nets import NetSpec, pool_out

ru4 = lambda x: K.round_up(int(x), 4)  # noqa: E731


@dataclass
class Act:
    spatial: bool
    c: int = 0        # channels (spatial) or features (flat)
    n: int = 0        # spatial size
    cs: int = 0       # pixel stride (spatial) or row stride (flat)
    fused_relu: bool = False
    value: torch.Tensor | None = None
    grad: torch.Tensor | None = None
    ones: bool = False  # flat: column c holds 1.0 (the FC weight-gradient GEMM's bias row)

    def shape(self, b):
        return (b, self.n, self.n, self.cs) if self.spatial else (b, self.cs)


@dataclass
class Op:
    kind: str
    layer: object
    inp: Act
    out: Act
    woff: int = -1
    wsz: int = 0
    boff: int = -1
    relu: bool = False
    first_param_layer: bool = False
    # conv
    c_in: int = 0
    k: int = 0
    s: int = 1
    p: int = 0
    m: int = 0
    Kc: int = 0
    Kf: int = 0
    ldK: int = 0
    ldW: int = 0     # row pitch of the weight-gradient staging (room for the bias column)
    wgrad_op: int = 1  # implicit layers: _abi.CONV_WGRAD, or CONV_WGRAD_BIAS (bias row folded in)
    w_inplace: bool = False
    implicit: bool = False
    s2d: tuple | None = None          # (stride, k2, pad2, n2, cp) of the space-to-depth form
    s2d_buf: torch.Tensor | None = None
    window: bool = False              # s2d layer on the window kernels (conv_window.cu, cp = 48)
    ldF: int = 0
    wflip: torch.Tensor | None = None
    dhat: torch.Tensor | None = None
    wstage: torch.Tensor | None = None
    dwstage: torch.Tensor | None = None
    # pool
    argmax: torch.Tensor | None = None
    # fc
    f_in: int = 0
    flat: Act | None = None
    extra: dict = field(default_factory=dict)


class GpuNet:
    """Device buffers + launch sequence for one NetSpec at a fixed max batch."""

    def __init__(self, net: NetSpec, batch: int, device=None, precision: str = "tf32",
                 explicit_only: bool = False, input_grad: bool = False, input_cs: int | None = None):
        if precision not in ("tf32", "3xtf32"):
            raise ValueError("precision must be 'tf32' or '3xtf32'")
        self.net = net
        self.b = int(batch)
        self.device = torch.device(device if device is not None else "cuda")
        self.prec = _abi.PRECISIONS[precision]
        self.precision = precision
        _abi.load()  # fail loudly now if the native library is missing
        z = lambda *shape, dtype=torch.float32: torch.zeros(shape, dtype=dtype, device=self.device)  # noqa: E731
        self._zeros = z
        geom = net.geometry()
        c0 = net.in_channels
        cs0 = c0 if input_cs is None else int(input_cs)   # pixel stride of the input
        if cs0 < c0:
            raise ValueError(f"input_cs {cs0} < channels {c0}")
        self.input = Act(True, c0, net.in_size, cs0)
        self.input.value = z(self.b, net.in_size, net.in_size, cs0)
        self.labels = z(self.b, dtype=torch.int32)
        self.ops: list[Op] = []
        cur = self.input
        # input_grad: the gradient w.r.t. the input is needed too (the merged-FC
        # head, whose input is the conv part's pool5 activation), so no layer is
        # treated as the first parameter layer (that one skips its data gradient)
        first_param = not input_grad
        i = 0
        while i < len(geom):
            g = geom[i]
            L = g.layer
            nxt_relu = i + 1 < len(geom) and geom[i + 1].layer.kind == "relu"
            if L.kind == "conv":
                c, n, _ = g.in_shape
                d, m, _ = g.out_shape
                out = Act(True, d, m, ru4(d), fused_relu=nxt_relu)
                op = Op("conv", L, cur, out, woff=g.param_offsets[0], wsz=g.param_sizes[0],
                        boff=g.param_offsets[1], relu=nxt_relu, first_param_layer=first_param,
                        c_in=c, k=L.k, s=L.stride, p=L.pad, m=m)
                op.Kc = c * L.k * L.k
                # Implicit GEMM (TMA im2col straight from the NHWC activation, no
                # lowered matrix) when the channels tile into 32-wide K blocks; the
                # data gradient then runs as a forward conv of dY with the flipped
                # kernel, which needs stride 1 and d_out % 32 == 0.
                op.implicit = (c % 32 == 0 and cur.cs % 4 == 0 and not explicit_only and
                               (first_param or (L.stride == 1 and d % 32 == 0)))
                # Strided first layer with few channels (CaffeNet conv1: 3 ch, k=11, s=4):
                # space-to-depth turns it into a stride-1 ceil(k/s)^2 conv over s*s*c
                # channels (padded to 32), i.e. another implicit GEMM.
                if (first_param and not op.implicit and not explicit_only and L.stride > 1
                        and L.pad % L.stride == 0):
                    st = L.stride
                    k2 = -(-L.k // st)
                    n2 = -(-n // st)
                    p2 = L.pad // st
                    cp = K.round_up(st * st * c, 32)
                    # the window kernels (TF32): no channel padding (cp = 48 for
                    # CaffeNet conv1), every tap read from one staged window per tile
                    window = (precision == "tf32" and p2 == 0 and st * st * c == 48 and
                              not os.environ.get("OMNI_NO_WINDOW") and
                              K.conv_window_plan(_abi.CONV_FPROP, self.b, n2, 48, k2, d) >= 0 and
                              K.conv_window_plan(_abi.CONV_WGRAD_BIAS, self.b, n2, 48, k2, d) >= 0)
                    if window:
                        cp = 48
                    if n2 + 2 * p2 - k2 + 1 == m and cp <= 2 * st * st * c:
                        op.s2d = (st, k2, p2, n2, cp)
                        op.implicit = True
                        op.window = window
                        # 64 floats of slack: the window wgrad's overlapping-row view
                        # of the image reads 16 floats past its last pixel
                        npx = self.b * n2 * n2 * cp
                        op.s2d_buf = z(npx + 64)[:npx].view(self.b, n2, n2, cp)
                if op.s2d is not None:
                    st, k2, p2, n2, cp = op.s2d
                    op.Kc = op.Kf = k2 * k2 * cp
                    op.ldK = K.round_up(op.Kf, 32)
                elif op.implicit:
                    op.Kf = op.Kc
                    op.ldK = K.round_up(op.Kf, 32)
                    if not first_param:
                        op.ldF = K.round_up(d * L.k * L.k, 32)
                        op.wflip = z(c, op.ldF)
                else:
                    # bias folded into the GEMM: ones column Kc in Dhat, bias in column Kc of W
                    op.Kf = op.Kc + (1 if op.boff >= 0 else 0)
                    # 128-byte row pitch: TMA boxes and TMA-stored rows stay line-aligned
                    op.ldK = K.round_up(op.Kf, 32)
                    op.dhat = z(self.b * m * m, op.ldK)
                op.wstage = z(d, op.ldK)
                op.ldW = op.ldK
                if op.window:
                    # weight + bias gradient on the window wgrad kernel: 48-wide tap
                    # rows, the bias in column k2*k2*48
                    st, k2, p2, n2, cp = op.s2d
                    op.wgrad_op = _abi.CONV_WGRAD_BIAS
                    op.ldW = K.round_up(k2 * k2 * cp + 4, 32)
                elif op.implicit and op.boff >= 0 and not os.environ.get("OMNI_NO_WGRAD_BIAS"):
                    # bias gradient as one more row of the implicit wgrad GEMM (column Kf)
                    op.wgrad_op = _abi.CONV_WGRAD_BIAS
                    op.ldW = K.round_up(op.Kf + 1, 32)
                op.dwstage = z(d, op.ldW)
                first_param = False
                i += 2 if nxt_relu else 1
            elif L.kind == "fc":
                f = int(torch.tensor(g.in_shape).prod())
                # row pitch with room for a ones column (the next FC layer's bias gradient)
                out = Act(False, L.d_out, 0, ru4(L.d_out + 1), fused_relu=nxt_relu)
                op = Op("fc", L, cur, out, woff=g.param_offsets[0], wsz=g.param_sizes[0],
                        boff=g.param_offsets[1], relu=nxt_relu, first_param_layer=first_param, f_in=f)
                if cur.spatial:
                    op.flat = Act(False, f, 0, ru4(f + 1), fused_relu=cur.fused_relu)
                    op.flat.value = z(self.b, op.flat.cs)
                    op.flat.value[:, f] = 1.0
                    op.flat.ones = True
                else:
                    op.flat = cur
                # FC weights (in, out) serve directly as the GEMM's B operand
                # (MN-major forward, K-major data gradient) when TMA can read them.
                op.w_inplace = L.d_out % 4 == 0 and g.param_offsets[0] % 4 == 0
                op.wstage = None if op.w_inplace else z(L.d_out, op.flat.cs)
                first_param = False
                i += 2 if nxt_relu else 1
            elif L.kind == "pool":
                c, n, _ = g.in_shape
                _, o, _ = g.out_shape
                out = Act(True, c, o, cur.cs)
                op = Op("pool", L, cur, out, k=L.k, s=L.stride or L.k, p=L.pad, m=o)
                if L.mode == "max":
                    op.argmax = z(self.b * o * o * c, dtype=torch.int32)
                i += 1
            elif L.kind == "relu":
                out = Act(cur.spatial, cur.c, cur.n, cur.cs)
                op = Op("relu", L, cur, out)
                i += 1
            else:  # pragma: no cover
                raise ValueError(L)
            out.value = z(*out.shape(self.b))
            if not out.spatial and out.cs > out.c:
                out.value[:, out.c] = 1.0   # never written by the GEMMs (N = c); ReLU keeps it 1
                out.ones = True
            self.ops.append(op)
            cur = out
        self.logits = cur
        # gradient buffers (the input needs none)
        for op in self.ops:
            op.out.grad = z(*op.out.shape(self.b))
            if op.kind == "fc" and op.flat is not op.inp and not op.first_param_layer:
                op.flat.grad = z(self.b, op.flat.cs)
        if input_grad:
            self.input.grad = z(*self.input.shape(self.b))
        self.first_fc = next((i for i, op in enumerate(self.ops) if op.kind == "fc"), len(self.ops))
        self.loss_buf = z(1)
        self.dim = net.dim
        self.grad = z(self.dim)
        self.wread = None
        # workspaces sized for the largest GEMM / bias reduction
        ws, bws, dd = 0, 0, 0
        for op in self.ops:
            ws = max(ws, self._workspace_need(op, self.b))
            if op.kind == "fc" and op.boff >= 0:
                bws = max(bws, K.bias_grad_ws_elems(self.b, op.layer.d_out))
            if op.kind == "conv" and op.implicit and op.boff >= 0:
                bws = max(bws, K.bias_grad_ws_elems(self.b * op.m * op.m, op.layer.d_out))
            if op.kind == "conv" and not op.first_param_layer and not op.implicit:
                dd = max(dd, self.b * op.m * op.m * op.ldK)
        self.gemm_ws = z(max(ws // 4, 4))
        self.gemm_ws_side = z(max(ws // 4, 4))   # weight-gradient GEMMs run on a side stream
        self._ws_active = self.gemm_ws
        self._s2d_ready = 0   # batch size whose space-to-depth input gather_batch wrote
        self._staged_for = None   # W whose layouts prestage() put in flight
        self.upd_stream = torch.cuda.Stream(device=self.device)   # layer-wise updates (backward(update=...))
        self._staged_ev = None
        self.side_stream = torch.cuda.Stream(device=self.device)
        self.bias_ws = z(max(bws, 4))
        self.ddhat = z(max(dd, 4))
        self.graph = None
        self.timer = None   # list -> (M, N, K, kind, ev0, ev1) per GEMM launch
        # False: weight gradients on the main stream (isolated kernel timing / debugging)
        self.overlap = not os.environ.get("OMNI_NO_SIDE_STREAM")
        # max pools over a fused-ReLU activation: mask folded into the argmax (mode 2)
        self.mark_pool = not os.environ.get("OMNI_NO_POOL_MARK")
        # FC bias gradients as one more row of the weight-gradient GEMM (the ones column)
        self.fc_bias_row = not os.environ.get("OMNI_NO_FC_BIAS_ROW")

    # ------------------------------------------------------------ shapes --
    def _workspace_need(self, op: Op, b: int) -> int:
        """Largest split-K workspace any GEMM of this layer asks for, from the
        same plan functions the launches use (implicit convs plan differently
        from plain GEMMs: 64-deep wgrad stages, transposed fprop)."""
        if op.kind == "conv" and op.implicit:
            d = op.layer.d_out
            if op.s2d is not None:
                st, k2, p2, n2, cp = op.s2d
                geo = (b, n2, cp, k2, 1, p2, d)
            else:
                geo = (b, op.inp.n, op.c_in, op.k, op.s, op.p, d)
            need = max(K.conv_implicit_workspace_bytes(self.prec, _abi.CONV_FPROP, *geo),
                       K.conv_implicit_workspace_bytes(self.prec, op.wgrad_op, *geo))
            if op.window:
                st, k2, p2, n2, cp = op.s2d
                need = max(need, K.conv_window_plan(_abi.CONV_WGRAD_BIAS, b, n2, cp, k2, d))
            if not op.first_param_layer:
                need = max(need, K.conv_implicit_workspace_bytes(
                    self.prec, _abi.CONV_FPROP, b, op.m, d, op.k, 1, op.k - 1 - op.p, op.c_in))
            return need
        return max([K.gemm_workspace_bytes(self.prec, M, N, Kd, False, False)
                    for M, N, Kd in self._gemm_shapes(op, b)] or [0])

    @staticmethod
    def _gemm_shapes(op: Op, b: int):
        if op.kind == "conv":
            Mr = b * op.m * op.m
            d = op.layer.d_out
            out = [(Mr, d, op.Kf), (d, op.Kf, Mr)]
            if not op.first_param_layer:
                if op.implicit:
                    out.append((b * op.inp.n * op.inp.n, op.c_in, d * op.k * op.k))
                else:
                    out.append((Mr, op.Kc, d))
            return out
        if op.kind == "fc":
            d = op.layer.d_out
            out = [(b, d, op.f_in), (op.f_in, d, b), (op.f_in + 1, d, b)]
            if not op.first_param_layer:
                out.append((b, op.f_in, d))
            return out
        return []

    def _timed(self, M, N, Kd, kind, fn):
        if self.timer is None:
            fn()
            return
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        self.timer.append((M, N, Kd, kind, e0, e1))

    def _gemm(self, M, N, Kd, A, lda, a_mn, B, ldb, b_mn, C, ldc, epi=_abi.EPI_STORE, bias=None,
              aux=None, ld_aux=0, kind="gemm"):
        self._timed(M, N, Kd, kind, lambda: K.gemm(
            M, N, Kd, A, lda, a_mn, B, ldb, b_mn, C, ldc, precision=self.prec, epilogue=epi,
            bias=bias, aux=aux, ld_aux=ld_aux, workspace=self._ws_active))

    def _conv_input(self, op, b, transform=True):
        """Activation + geometry the implicit GEMM of a conv layer reads: the layer
        input itself, or its space-to-depth form (built here in forward)."""
        if op.s2d is None:
            return op.inp.value[:b], op.c_in, op.k, op.s, op.p
        st, k2, p2, n2, cp = op.s2d
        if transform:
            if self._s2d_ready == b and op.inp is self.input:
                self._s2d_ready = 0          # written by the fused gather
            else:
                K.space_to_depth(op.inp.value[:b], op.c_in, st, op.s2d_buf[:b])
        return op.s2d_buf[:b], cp, k2, 1, p2

    def _conv(self, op_code, X, c, k, s, p, d, G, ldg, Y, ldy, epi=_abi.EPI_STORE, bias=None,
              aux=None, ld_aux=0):
        b, n = X.shape[0], X.shape[1]
        m = (n + 2 * p - k) // s + 1
        if op_code == _abi.CONV_FPROP:
            M, N, Kd = b * m * m, d, c * k * k
        else:   # (the bias row of CONV_WGRAD_BIAS is not counted as conv work)
            M, N, Kd = d, c * k * k, b * m * m
        self._timed(M, N, Kd, "conv", lambda: K.conv_implicit(
            op_code, X, c, k, s, p, d, G, ldg, Y, ldy, precision=self.prec, epilogue=epi,
            bias=bias, aux=aux, ld_aux=ld_aux, workspace=self._ws_active))

    # ----------------------------------------------------------- staging --
    def stage_weights(self, W: torch.Tensor) -> None:
        """Flat fp32 parameters -> GEMM-ready layouts (tap-major conv rows with the
        bias in column Kc; transposed FC weights only when they cannot be used in place)."""
        if W.data_ptr() % 16:
            raise ValueError("the flat parameter vector must be 16-byte aligned")
        self._W = W
        for op in self.ops:
            if op.kind == "conv" and op.s2d is not None:
                st, k2, p2, n2, cp = op.s2d
                K.conv_weight_s2d(W[op.woff:op.woff + op.wsz], op.layer.d_out, op.c_in, op.k, st,
                                  cp, op.wstage, op.ldK)
            elif op.kind == "conv":
                d = op.layer.d_out
                bias = W[op.boff:op.boff + d] if op.boff >= 0 and not op.implicit else None
                K.conv_weight_to_tap(W[op.woff:op.woff + op.wsz], d, op.c_in, op.k, op.wstage,
                                     op.ldK, bias=bias)
                if op.wflip is not None:
                    K.conv_weight_flip(W[op.woff:op.woff + op.wsz], d, op.c_in, op.k, op.wflip,
                                       op.ldF)
            elif op.kind == "fc" and not op.w_inplace:
                d = op.layer.d_out
                K.transpose(W[op.woff:op.woff + op.wsz], d, 0, op.f_in, d, op.wstage, op.flat.cs, 0, 1)

    def prestage(self, W: torch.Tensor) -> None:
        """Stage W's layouts on the side stream, after the main stream's pending
        work (the previous update), so they overlap whatever the main stream
        does next (the batch gather); forward(W) then only waits for them."""
        if not self.overlap:
            return
        main = torch.cuda.current_stream(self.device)
        ev = torch.cuda.Event()
        ev.record(main)
        self.side_stream.wait_event(ev)
        with torch.cuda.stream(self.side_stream):
            self.stage_weights(W)
            self._staged_ev = torch.cuda.Event()
            self._staged_ev.record(self.side_stream)
        self._staged_for = W

    # ----------------------------------------------------------- forward --
    def forward(self, W: torch.Tensor, b: int | None = None, need_grad: bool = True,
                stop: int | None = None) -> torch.Tensor:
        """Run the forward pass on self.input / self.labels (first b rows);
        leaves the mean loss in self.loss_buf and, if need_grad, dlogits in
        the logits' grad buffer.  W is the flat fp32 parameter vector.
        ``stop``: run ops[:stop] only (the conv part of a merged-FC mapping; no
        loss) -- the activation then waits in ops[stop].inp.value."""
        b = self.b if b is None else int(b)
        staged = self._staged_for
        self._staged_for = None
        if staged is not None:
            torch.cuda.current_stream(self.device).wait_event(self._staged_ev)
        if staged is None or staged is not W:
            self.stage_weights(W)
        for op in (self.ops if stop is None else self.ops[:stop]):
            L = op.layer
            if op.kind == "conv":
                d = L.d_out
                Mr = b * op.m * op.m
                if op.implicit:
                    if op.boff >= 0:
                        epi = _abi.EPI_BIAS_RELU if op.relu else _abi.EPI_BIAS
                        bias = W[op.boff:op.boff + d]
                    else:
                        epi = _abi.EPI_RELU if op.relu else _abi.EPI_STORE
                        bias = None
                    X, c_, k_, s_, p_ = self._conv_input(op, b)
                    if op.window:
                        self._timed(Mr, d, op.c_in * op.k * op.k, "conv", lambda: K.conv_window(
                            _abi.CONV_FPROP, X, k_, d, op.wstage, op.ldK, op.out.value, op.out.cs,
                            epilogue=epi, bias=bias))
                        continue
                    self._conv(_abi.CONV_FPROP, X, c_, k_, s_, p_, d, op.wstage, op.ldK,
                               op.out.value, op.out.cs, epi, bias)
                    continue
                K.lower_nhwc(op.inp.value[:b], op.c_in, op.k, op.s, op.p, op.ldK, out=op.dhat,
                             ones_col=op.boff >= 0)
                epi = _abi.EPI_RELU if op.relu else _abi.EPI_STORE
                self._gemm(Mr, d, op.Kf, op.dhat, op.ldK, False, op.wstage, op.ldK, False,
                           op.out.value, op.out.cs, epi, kind="conv")
            elif op.kind == "pool":
                mode = 0 if L.mode == "max" else 1
                if mode == 0 and op.inp.fused_relu and self.mark_pool:
                    mode = 2   # the ReLU mask of the routed element folded into the argmax
                K.pool_fwd(mode, op.inp.value[:b], op.inp.c, op.k, op.s, op.p, L.ceil,
                           op.out.value[:b], op.argmax)
            elif op.kind == "relu":
                n = b * (op.out.value[0].numel())
                K.relu_fwd(op.inp.value.view(-1)[:n], op.out.value.view(-1)[:n])
            elif op.kind == "fc":
                d = L.d_out
                if op.flat is not op.inp:
                    hw = op.inp.n * op.inp.n
                    K.transpose(op.inp.value, op.inp.cs, hw * op.inp.cs, hw, op.inp.c,
                                op.flat.value, hw, op.flat.cs, b)
                if op.boff >= 0:
                    epi = _abi.EPI_BIAS_RELU if op.relu else _abi.EPI_BIAS
                    bias = W[op.boff:op.boff + d]
                else:
                    epi = _abi.EPI_RELU if op.relu else _abi.EPI_STORE
                    bias = None
                if op.w_inplace:
                    self._gemm(b, d, op.f_in, op.flat.value, op.flat.cs, False,
                               W[op.woff:op.woff + op.wsz], d, True, op.out.value, op.out.cs, epi, bias)
                else:
                    self._gemm(b, d, op.f_in, op.flat.value, op.flat.cs, False, op.wstage,
                               op.flat.cs, False, op.out.value, op.out.cs, epi, bias)
        if stop is not None:
            return None
        C = self.net.classes
        K.softmax_xent(self.logits.value, self.logits.cs, self.labels, b, C, self.loss_buf,
                       self.logits.grad if need_grad else None, self.logits.cs, 1.0 / b)
        return self.loss_buf

    # ---------------------------------------------------------- backward --
    def backward(self, b: int | None = None, on_grad=None, update=None,
                 start: int | None = None, fused_update=None) -> torch.Tensor:
        """Gradient of the mean loss w.r.t. the flat parameters -> self.grad.

        ``on_grad(lo, hi)`` (optional) is called as soon as the launches that
        write G[lo:hi] (one layer's weight + bias gradient) are enqueued, in
        backward order -- the hook a data-parallel caller uses to overlap the
        gradient allreduce of finished layers with the rest of the backward; if
        it returns an async work handle, that layer's update waits for it.

        ``update = (W, V, w_read, eta, mu, lam)`` (single device) applies the
        momentum update (K8) layer by layer as soon as a layer's gradient is
        final and its data gradient no longer needs W, on a third stream: the
        FC layers' update (94% of CaffeNet's parameters) overlaps the conv
        backward instead of ending the step.

        ``start``: back-propagate through ops[:start] only, from the gradient
        already placed in ops[start].inp.grad (merged-FC conv part).

        ``fused_update(lo, hi, stream)`` (with ``update``) replaces the layer's
        allreduce + update: it is called on the update stream once G[lo:hi] is
        final and W[lo:hi] is no longer read (peer-memory data parallelism,
        ``comm.PeerUpdate``)."""
        b = self.b if b is None else int(b)
        G = self.grad
        main = torch.cuda.current_stream(self.device)
        side = self.side_stream
        net = self
        pending = []   # [(lo, hi, event after the layer's weight gradient)]

        def done(op):
            hi = op.boff + op.layer.d_out if op.boff >= 0 else op.woff + op.wsz
            work = on_grad(op.woff, hi) if on_grad is not None else None
            if update is not None:
                ev = torch.cuda.Event()
                ev.record(torch.cuda.current_stream(self.device))   # after the wgrad launches
                pending.append((op.woff, hi, ev, work))

        def flush():
            """Issue the updates of layers whose data gradient is enqueued."""
            if update is None or not pending:
                return
            Wu, Vu, wr, eta, mu, lam = update
            us = self.upd_stream if self.overlap else main
            ev_main = torch.cuda.Event()
            ev_main.record(main)                                     # the dgrads read W in place
            us.wait_event(ev_main)
            for lo, hi, ev, work in pending:
                us.wait_event(ev)
                with torch.cuda.stream(us):
                    if fused_update is not None:
                        fused_update(lo, hi, us)
                        continue
                    if work is not None:
                        work.wait()      # this layer's gradient allreduce (update stream waits)
                    K.sgd_momentum(Wu[lo:hi], Vu[lo:hi], G[lo:hi], wr[lo:hi], eta, mu, lam)
            pending.clear()

        class wgrad_stream:
            """Weight/bias gradients only feed the update, so they run on a side
            stream (own split-K workspace) while the data-gradient chain continues
            on the main stream; joined at the end of backward."""

            def __enter__(self):
                ev = torch.cuda.Event()
                ev.record(main)
                side.wait_event(ev)
                self.ctx = torch.cuda.stream(side if net.overlap else main)
                self.ctx.__enter__()
                net._ws_active = net.gemm_ws_side

            def __exit__(self, *exc):
                net._ws_active = net.gemm_ws
                return self.ctx.__exit__(*exc)

        for op in reversed(self.ops if start is None else self.ops[:start]):
            flush()
            L = op.layer
            if op.kind == "fc":
                d = L.d_out
                dZ = op.out.grad
                with wgrad_stream():
                    if op.boff == op.woff + op.wsz and op.flat.ones and self.fc_bias_row:
                        # weight + bias gradient in one GEMM: the input's ones column is
                        # row f of X^T, and the bias follows the (in, out) weights in G
                        self._gemm(op.f_in + 1, d, b, op.flat.value, op.flat.cs, True, dZ, op.out.cs,
                                   True, G[op.woff:op.boff + d], d)
                    else:
                        # weight gradient straight into the flat (in, out) slice
                        self._gemm(op.f_in, d, b, op.flat.value, op.flat.cs, True, dZ, op.out.cs, True,
                                   G[op.woff:op.woff + op.wsz], d)
                        if op.boff >= 0:
                            K.bias_grad(dZ, op.out.cs, b, d, G[op.boff:op.boff + d], self.bias_ws)
                    done(op)
                if op.first_param_layer:
                    continue
                if op.w_inplace:   # B(j=f, r=o) = W[f*d + o]: K-major, ld = d
                    Bop, ldb, bmn = self._W[op.woff:op.woff + op.wsz], d, False
                else:              # B(j=f, r=o) = Wt[o*ld_in + f]: MN-major
                    Bop, ldb, bmn = op.wstage, op.flat.cs, True
                if op.flat is op.inp:
                    if op.inp.fused_relu:
                        self._gemm(b, op.f_in, d, dZ, op.out.cs, False, Bop, ldb, bmn,
                                   op.inp.grad, op.inp.cs, _abi.EPI_MASK_AUX, aux=op.inp.value,
                                   ld_aux=op.inp.cs)
                    else:
                        self._gemm(b, op.f_in, d, dZ, op.out.cs, False, Bop, ldb, bmn,
                                   op.inp.grad, op.inp.cs)
                else:
                    self._gemm(b, op.f_in, d, dZ, op.out.cs, False, Bop, ldb, bmn,
                               op.flat.grad, op.flat.cs)
                    hw = op.inp.n * op.inp.n
                    K.transpose(op.flat.grad, hw, op.flat.cs, op.inp.c, hw, op.inp.grad,
                                op.inp.cs, hw * op.inp.cs, b)
                    if op.inp.fused_relu:
                        n = b * op.inp.grad[0].numel()
                        K.relu_bwd(op.inp.grad.view(-1)[:n], op.inp.value.view(-1)[:n],
                                   op.inp.grad.view(-1)[:n])
            elif op.kind == "conv":
                d = L.d_out
                Mr = b * op.m * op.m
                dZ = op.out.grad
                if op.implicit:
                    with wgrad_stream():
                        X, c_, k_, s_, p_ = self._conv_input(op, b, transform=False)
                        if op.window:
                            self._timed(d, c_ * k_ * k_, Mr, "conv", lambda: K.conv_window(
                                _abi.CONV_WGRAD_BIAS, X, k_, d, dZ, op.out.cs, op.dwstage, op.ldW,
                                workspace=self._ws_active))
                        else:
                            self._conv(op.wgrad_op, X, c_, k_, s_, p_, d, dZ, op.out.cs,
                                       op.dwstage, op.ldW)
                        fold = op.wgrad_op == _abi.CONV_WGRAD_BIAS
                        gb = G[op.boff:op.boff + d] if fold else None
                        if op.s2d is not None:
                            # wgrad rows are cp (window kernel) or round_up(cp, 32) wide per tap
                            cpw = op.s2d[4] if op.window else K.round_up(op.s2d[4], 32)
                            K.conv_weight_s2d(G[op.woff:op.woff + op.wsz], d, op.c_in, op.k,
                                              op.s2d[0], cpw, op.dwstage, op.ldW,
                                              inverse=True, bias=gb)
                        else:
                            K.conv_weight_to_tap(G[op.woff:op.woff + op.wsz], d, op.c_in, op.k,
                                                 op.dwstage, op.ldW, inverse=True, bias=gb)
                        if op.boff >= 0 and not fold:
                            K.bias_grad(dZ, op.out.cs, Mr, d, G[op.boff:op.boff + d], self.bias_ws)
                        done(op)
                    if op.first_param_layer:
                        continue
                    # dX = conv(dY, flipped kernel, pad k-1-p) with the ReLU mask of X fused
                    if op.inp.fused_relu:
                        self._conv(_abi.CONV_FPROP, dZ[:b], d, op.k, 1, op.k - 1 - op.p, op.c_in,
                                   op.wflip, op.ldF, op.inp.grad, op.inp.cs, _abi.EPI_MASK_AUX,
                                   aux=op.inp.value, ld_aux=op.inp.cs)
                    else:
                        self._conv(_abi.CONV_FPROP, dZ[:b], d, op.k, 1, op.k - 1 - op.p, op.c_in,
                                   op.wflip, op.ldF, op.inp.grad, op.inp.cs)
                    continue
                with wgrad_stream():
                    # weight (and, via the ones column, bias) gradient in one GEMM
                    self._gemm(d, op.Kf, Mr, dZ, op.out.cs, True, op.dhat, op.ldK, True, op.dwstage,
                               op.ldK, kind="conv")
                    K.conv_weight_to_tap(G[op.woff:op.woff + op.wsz], d, op.c_in, op.k, op.dwstage,
                                         op.ldK, inverse=True,
                                         bias=G[op.boff:op.boff + d] if op.boff >= 0 else None)
                    done(op)
                if op.first_param_layer:
                    continue
                self._gemm(Mr, op.Kc, d, dZ, op.out.cs, False, op.wstage, op.ldK, True, self.ddhat,
                           op.ldK, kind="conv")
                K.col2im_nhwc(self.ddhat, op.ldK, b, op.inp.n, op.c_in, op.inp.cs, op.k, op.s, op.p,
                              op.inp.grad, op.inp.value if op.inp.fused_relu else None)
            elif op.kind == "pool":
                if op.inp.grad is None:
                    continue
                mode = 0 if L.mode == "max" else 1
                if mode == 0 and op.inp.fused_relu and self.mark_pool:
                    # max pool: forward mode 2 marked the windows whose max is not > 0
                    xm, rm = None, 0
                elif mode == 0 and op.inp.fused_relu:
                    # max pool: the ReLU mask of the routed element is (pooled value > 0)
                    xm, rm = op.out.value[:b], 2
                else:
                    xm, rm = op.inp.value, int(op.inp.fused_relu)
                K.pool_bwd(mode, op.out.grad[:b], (b, op.inp.n, op.inp.n, op.inp.cs), op.inp.c,
                           op.k, op.s, op.p, L.ceil, op.argmax, xm, rm, op.inp.grad)
            elif op.kind == "relu":
                if op.inp.grad is None:
                    continue
                n = b * op.out.grad[0].numel()
                K.relu_bwd(op.out.grad.view(-1)[:n], op.out.value.view(-1)[:n],
                           op.inp.grad.view(-1)[:n])
        flush()
        main.wait_stream(side)
        if update is not None and self.overlap:
            main.wait_stream(self.upd_stream)
        return G

    # ------------------------------------------------------------- input --
    def load_batch(self, X_nhwc: torch.Tensor, y: torch.Tensor) -> None:
        b = X_nhwc.shape[0]
        self._s2d_ready = 0
        self.input.value[:b].copy_(X_nhwc)
        self.labels[:b].copy_(y)

    def gather_batch(self, data: torch.Tensor, labels: torch.Tensor, idx: torch.Tensor) -> None:
        """Device gather of a sampled batch (problems.py:197-199) from a
        device-resident NHWC dataset.  When the first layer runs on the
        space-to-depth form of the input, the gather writes that form directly
        (one fused pass; the raw input buffer is not materialised)."""
        first = self.ops[0] if self.ops else None
        if (first is not None and first.kind == "conv" and first.s2d is not None
                and first.inp is self.input and idx.dtype == torch.int64):
            K.space_to_depth_gather(data, idx, first.c_in, first.s2d[0],
                                    first.s2d_buf[:idx.numel()])
            self._s2d_ready = idx.numel()
        else:
            K.gather_rows(data, idx, self.input.value)
        K.gather_i32(labels, idx, self.labels)

    def loss_and_grad(self, W: torch.Tensor, b: int | None = None):
        self.forward(W, b, need_grad=True)
        self.backward(b)
        return self.loss_buf, self.grad

