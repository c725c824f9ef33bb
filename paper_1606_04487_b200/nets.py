"""Network specifications: the layer lists the benchmark configs name.

The reference has exactly one CNN, ``TinyCNNProblem`` (problems.py:152-275:
conv 3x3 pad 1 1->4, ReLU, 2x2/2 max-pool, linear, softmax-CE, no bias).
``NetSpec`` generalises it to the layer vocabulary of the paper's networks
 -- conv, ReLU, max/avg pooling with Caffe's ceil rule,
fully connected -- keeping the reference's parameter packing rule
(problems.py:201-204): one flat vector, layer by layer, weight before bias,
C order; conv weights (d_out, d_in, k, k), FC weights (in, out) with the
input flattened in (c, h, w) order.

Deviations from the Caffe prototxts, documented once here: LRN and dropout
are SPEC non-goals and are omitted; CaffeNet is ungrouped
(PAPER.md:2099).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np


@dataclass(frozen=True)
class Conv:
    d_out: int
    k: int
    stride: int = 1
    pad: int = 0
    bias: bool = True
    kind: str = field(default="conv", init=False)


@dataclass(frozen=True)
class ReLU:
    kind: str = field(default="relu", init=False)


@dataclass(frozen=True)
class Pool:
    k: int
    stride: Optional[int] = None
    pad: int = 0
    mode: str = "max"
    ceil: bool = True
    kind: str = field(default="pool", init=False)

    def __post_init__(self) -> None:
        if self.mode not in ("max", "avg"):
            raise ValueError(f"unknown pooling mode {self.mode!r}")


@dataclass(frozen=True)
class FC:
    d_out: int
    bias: bool = True
    kind: str = field(default="fc", init=False)


def conv_out(n: int, k: int, s: int, p: int) -> int:
    if min(n, k, s) < 1 or p < 0:
        raise ValueError("n, k, d_in, d_out, stride must be positive")
    if k > n + 2 * p:
        raise ValueError(f"kernel {k} exceeds padded input {n + 2 * p}")
    span = n + 2 * p - k
    if span % s:
        raise ValueError(
            f"output size not integral: (n + 2*pad - k) = {span} is not divisible by stride {s}"
        )
    return span // s + 1


def pool_out(n: int, k: int, s: int, p: int, ceil_mode: bool) -> int:
    span = n + 2 * p - k
    out = (-(-span // s) if ceil_mode else span // s) + 1
    if p > 0 and (out - 1) * s >= n + p:
        out -= 1
    return out


@dataclass(frozen=True)
class LayerGeom:
    index: int
    layer: object
    in_shape: tuple   # (c, n, n) spatial or (f,) flat
    out_shape: tuple
    param_offsets: tuple  # (weight_off, bias_off or -1)
    param_sizes: tuple


@dataclass(frozen=True)
class NetSpec:
    """A feed-forward CNN ending in softmax cross-entropy."""

    name: str
    in_channels: int
    in_size: int
    layers: tuple
    classes: int = field(init=False)

    def __post_init__(self) -> None:
        if not self.layers or self.layers[-1].kind != "fc":
            raise ValueError("a NetSpec must end with a fully connected layer")
        object.__setattr__(self, "classes", self.layers[-1].d_out)
        self.geometry()  # validate

    def geometry(self) -> list[LayerGeom]:
        out = []
        cur = (self.in_channels, self.in_size, self.in_size)
        off = 0
        for i, L in enumerate(self.layers):
            if L.kind == "conv":
                if len(cur) != 3:
                    raise ValueError("conv after a fully connected layer")
                c, n, _ = cur
                m = conv_out(n, L.k, L.stride, L.pad)
                wsz = L.d_out * c * L.k * L.k
                bsz = L.d_out if L.bias else 0
                nxt = (L.d_out, m, m)
            elif L.kind == "pool":
                if len(cur) != 3:
                    raise ValueError("pooling after a fully connected layer")
                c, n, _ = cur
                s = L.stride or L.k
                if L.k > n + 2 * L.pad or L.pad >= L.k:
                    raise ValueError(f"invalid pooling window k={L.k} pad={L.pad} for n={n}")
                o = pool_out(n, L.k, s, L.pad, L.ceil)
                wsz = bsz = 0
                nxt = (c, o, o)
            elif L.kind == "relu":
                wsz = bsz = 0
                nxt = cur
            elif L.kind == "fc":
                f = int(np.prod(cur))
                wsz = f * L.d_out
                bsz = L.d_out if L.bias else 0
                nxt = (L.d_out,)
            else:
                raise ValueError(f"unknown layer {L!r}")
            woff = off
            boff = off + wsz if bsz else -1
            off += wsz + bsz
            out.append(LayerGeom(i, L, cur, nxt, (woff, boff), (wsz, bsz)))
            cur = nxt
        return out

    @property
    def dim(self) -> int:
        g = self.geometry()[-1]
        return (g.param_offsets[0] + sum(g.param_sizes)) if g.param_sizes else 0

    def to_dicts(self) -> list[dict]:
        """Plain-dict form (what the CPU oracle consumes)."""
        out = []
        for L in self.layers:
            if L.kind == "conv":
                out.append({"kind": "conv", "d_out": L.d_out, "k": L.k, "stride": L.stride,
                            "pad": L.pad, "bias": L.bias})
            elif L.kind == "relu":
                out.append({"kind": "relu"})
            elif L.kind == "pool":
                out.append({"kind": "pool", "mode": L.mode, "k": L.k, "stride": L.stride or L.k,
                            "pad": L.pad, "ceil": L.ceil})
            else:
                out.append({"kind": "fc", "d_out": L.d_out, "bias": L.bias})
        return out

    def conv_flops_per_image(self) -> float:
        """Conv GEMM FLOPs per image, FW + BW (wgrad + dgrad; no dgrad for the
        first layer), the accounting of PAPER.md:1822."""
        tot = 0.0
        first = True
        for g in self.geometry():
            if g.layer.kind == "conv":
                c, n, _ = g.in_shape
                d, m, _ = g.out_shape
                f = 2.0 * m * m * d * c * g.layer.k ** 2
                tot += f * (2 if first else 3)
                first = False
        return tot

    def fc_flops_per_image(self) -> float:
        tot = 0.0
        first_param = True
        for g in self.geometry():
            if g.layer.kind == "fc":
                f = 2.0 * int(np.prod(g.in_shape)) * g.layer.d_out
                tot += 3 * f
            if g.param_sizes[0]:
                first_param = False
        return tot


# ---------------------------------------------------------------- presets --
def tiny_cnn(image_size: int = 8, classes: int = 4) -> NetSpec:
    """The reference TinyCNN (problems.py:152-184)."""
    return NetSpec("tiny_cnn", 1, image_size, (
        Conv(4, 3, 1, 1, bias=False), ReLU(), Pool(2, 2, 0, "max", ceil=False),
        FC(classes, bias=False)))


def lenet() -> NetSpec:
    """Caffe LeNet (28x28x1, 10 classes)."""
    return NetSpec("lenet", 1, 28, (
        Conv(20, 5), Pool(2, 2), Conv(50, 5), Pool(2, 2), FC(500), ReLU(), FC(10)))


def cifar10_quick() -> NetSpec:
    """Caffe CIFAR-10 quick (32x32x3, 10 classes): max pool before ReLU in block 1,
    average pooling in blocks 2 and 3, ceil-mode pooling."""
    return NetSpec("cifar10_quick", 3, 32, (
        Conv(32, 5, 1, 2), Pool(3, 2), ReLU(),
        Conv(32, 5, 1, 2), ReLU(), Pool(3, 2, mode="avg"),
        Conv(64, 5, 1, 2), ReLU(), Pool(3, 2, mode="avg"),
        FC(64), FC(10)))


def caffenet() -> NetSpec:
    """CaffeNet / AlexNet (227x227x3, 1000 classes), ungrouped, no LRN/dropout."""
    return NetSpec("caffenet", 3, 227, (
        Conv(96, 11, 4, 0), ReLU(), Pool(3, 2),
        Conv(256, 5, 1, 2), ReLU(), Pool(3, 2),
        Conv(384, 3, 1, 1), ReLU(),
        Conv(384, 3, 1, 1), ReLU(),
        Conv(256, 3, 1, 1), ReLU(), Pool(3, 2),
        FC(4096), ReLU(), FC(4096), ReLU(), FC(1000)))


def vgg16() -> NetSpec:
    """VGG-16 (224x224x3, 1000 classes): 13 conv 3x3/1/1 + 5 max-pool 2/2 + 3 FC."""
    layers = []
    for d, reps in ((64, 2), (128, 2), (256, 3), (512, 3), (512, 3)):
        for _ in range(reps):
            layers += [Conv(d, 3, 1, 1), ReLU()]
        layers.append(Pool(2, 2))
    layers += [FC(4096), ReLU(), FC(4096), ReLU(), FC(1000)]
    return NetSpec("vgg16", 3, 224, tuple(layers))


PRESETS = {"tiny_cnn": tiny_cnn, "lenet": lenet, "cifar10_quick": cifar10_quick,
           "caffenet": caffenet, "vgg16": vgg16}


def get(name: str, **kw) -> NetSpec:
    try:
        return PRESETS[name](**kw)
    except KeyError:
        raise ValueError(f"unknown network {name!r}; choose from {sorted(PRESETS)}") from None


def fc_head(net: NetSpec) -> tuple[NetSpec, int]:
    """Split at the first fully connected layer (the merged-FC mapping,
    PAPER.md:936-959): returns the FC head as its own NetSpec, whose input is
    the conv part's last activation, and the flat-parameter offset where the
    head's parameters start (FC layers come last in the packing, so the head's
    parameter vector is W[offset:])."""
    geo = net.geometry()
    j = next((g.index for g in geo if g.layer.kind == "fc"), None)
    if j is None or len(geo[j].in_shape) != 3:
        raise ValueError("merged FC needs a conv part followed by fully connected layers")
    c, n, _ = geo[j].in_shape
    head = NetSpec(f"{net.name}_fc_head", c, n, tuple(net.layers[j:]))
    off = geo[j].param_offsets[0]
    if head.dim != net.dim - off:
        raise ValueError("FC head parameters are not the tail of the packing")
    return head, off
