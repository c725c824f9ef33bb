"""CPU ORACLE -- test infrastructure only, never the product path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module, and only as the checker (or as the
timed reference CPU implementation).  Nothing in paper_1606_04487_b200/ imports
it.

A float64 NumPy restatement of the reference's hot path (omnisim 0.1.0,
/root/reference/pkg/src/omnisim), extended -- from the same primitives -- to
the multi-layer networks the benchmark configs name:

* lowering / blocked GEMM / lifting / direct conv: tensors.py:144-256
* conv -> ReLU -> max-pool -> linear -> softmax-CE cascade and its hand-written
  backward: problems.py:206-269 (mean-over-batch gradient :248, strict ReLU
  mask :261, first-max pool routing :215-216, flat W packing :201-204)
* momentum SGD with a possibly stale snapshot: sgd.py:92-112
* RNG streams: sgd.py:28-46; the g-group event loop: simulator.py:123-213

Extensions the reference does not have (multi-layer, bias, k x k / s pooling
with Caffe's ceil rule, average pooling, FC stacks, conv input gradient via
col2im) are restated from the same primitives and pinned by the adjoint
identity and central finite differences in tests/test_oracle.py.  Parity of the
restatement itself is pinned against fixtures generated from the reference
(tests/golden/make_golden.py).
"""

from __future__ import annotations

import heapq
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

GEMM_BLOCK = 128  # tensors.py:28


# ------------------------------------------------------------ geometry ----
def conv_out(n: int, k: int, s: int, p: int) -> int:
    """m = (n + 2p - k)/s + 1 (tensors.py:57-59); same validity rules (:42-54)."""
    if min(n, k, s) < 1 or p < 0 or k > n + 2 * p or (n + 2 * p - k) % s:
        raise ValueError(f"invalid conv geometry n={n} k={k} s={s} p={p}")
    return (n + 2 * p - k) // s + 1


def pool_out(n: int, k: int, s: int, p: int, ceil_mode: bool) -> int:
    """Caffe's pooled size: ceil (or floor) of the span over stride, plus one,
    minus one if the last window would start in the right padding."""
    span = n + 2 * p - k
    out = (-(-span // s) if ceil_mode else span // s) + 1
    if p > 0 and (out - 1) * s >= n + p:
        out -= 1
    return out


# ---------------------------------------------------- tensors.py restated --
def lower(D: np.ndarray, k: int, s: int, p: int, start: int = 0, b_p: int | None = None):
    """D (b, c, n, n) -> Dhat (b_p*m^2, c*k*k): row = img*m^2 + x*m + y, column =
    (ch*k + kx)*k + ky, zero padding (tensors.py:164-181).  Built from explicit
    index arrays (a pure gather), so it is bit-exact with the reference."""
    b, c, n, _ = D.shape
    b_p = b if b_p is None else b_p
    m = conv_out(n, k, s, p)
    chunk = D[start:start + b_p]
    padded = np.zeros((b_p, c, n + 2 * p, n + 2 * p), dtype=D.dtype)
    padded[:, :, p:p + n, p:p + n] = chunk
    xs = (np.arange(m) * s)[:, None] + np.arange(k)[None, :]  # (m, k) padded row index
    rows = xs[:, None, :, None]                                 # x, -, kx, -
    cols = xs[None, :, None, :]                                 # -, y, -, ky
    g = padded[:, :, rows, cols]                                # (b_p, c, m, m, k, k)
    return np.ascontiguousarray(g.transpose(0, 2, 3, 1, 4, 5).reshape(b_p * m * m, c * k * k))


# "einsum": the reference's blocked einsum (tensors.py:193-210) -- what the CPU
# baseline times.  "blas": one float64 BLAS product per call; the summation order
# differs from the blocked einsum only at the 1e-16 level, which is far below
# every fp32 tolerance, so the large-batch parity tests (CaffeNet at b=256) use
# it to keep the checker to seconds.  Select with ``gemm_impl("blas")``.
GEMM_IMPL = "einsum"


class gemm_impl:
    """Context manager: ``with gemm_impl("blas"): ...`` (restores on exit)."""

    def __init__(self, name: str):
        if name not in ("einsum", "blas"):
            raise ValueError(name)
        self.name = name

    def __enter__(self):
        global GEMM_IMPL
        self.prev, GEMM_IMPL = GEMM_IMPL, self.name
        return self

    def __exit__(self, *exc):
        global GEMM_IMPL
        GEMM_IMPL = self.prev


def gemm(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """R = A @ B in float64 with the inner dimension consumed in ascending
    GEMM_BLOCK-wide blocks, one einsum per block (tensors.py:193-210)."""
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    if GEMM_IMPL == "blas":
        return A @ B
    out = np.zeros((A.shape[0], B.shape[1]))
    for j0 in range(0, A.shape[1], GEMM_BLOCK):
        j1 = min(j0 + GEMM_BLOCK, A.shape[1])
        out += np.einsum("ik,kj->ij", A[:, j0:j1], B[j0:j1, :])
    return out


def lower_kernel(K: np.ndarray) -> np.ndarray:
    """(d_out, d_in, k, k) -> (d_in*k*k, d_out) (tensors.py:184-190)."""
    return np.ascontiguousarray(K.reshape(K.shape[0], -1).T)


def lift(Rhat: np.ndarray, b: int, m: int, d_out: int) -> np.ndarray:
    """(b*m^2, d_out) -> NCHW (tensors.py:213-219)."""
    return np.ascontiguousarray(Rhat.reshape(b, m, m, d_out).transpose(0, 3, 1, 2))


def conv_lowered(D, K, s=1, p=0, b_p=None, workers=1):
    """lower -> gemm -> lift over contiguous batch partitions (tensors.py:222-256)."""
    b = D.shape[0]
    d_out, _, k, _ = K.shape
    m = conv_out(D.shape[2], k, s, p)
    b_p = b if b_p is None else b_p
    Khat = lower_kernel(K)
    Rhat = np.empty((b * m * m, d_out))
    bounds = np.linspace(0, b, num=min(workers, b) + 1, dtype=int)

    def part(lo, hi):
        for c0 in range(lo, hi, b_p):
            size = min(b_p, hi - c0)
            Rhat[c0 * m * m:(c0 + size) * m * m] = gemm(lower(D, k, s, p, c0, size), Khat)

    parts = [(int(a), int(z)) for a, z in zip(bounds[:-1], bounds[1:]) if z > a]
    if len(parts) == 1:
        part(*parts[0])
    else:
        with ThreadPoolExecutor(max_workers=len(parts)) as ex:
            list(ex.map(lambda ab: part(*ab), parts))
    return lift(Rhat, b, m, d_out)


def conv_direct(D, K, s=1, p=0):
    """Sliding-window accumulation over (kx, ky) (tensors.py:144-161)."""
    b = D.shape[0]
    d_out, _, k, _ = K.shape
    m = conv_out(D.shape[2], k, s, p)
    padded = np.pad(D, ((0, 0), (0, 0), (p, p), (p, p)))
    out = np.zeros((b, d_out, m, m))
    hi = s * (m - 1) + 1
    for kx in range(k):
        for ky in range(k):
            win = padded[:, :, kx:kx + hi:s, ky:ky + hi:s]
            out += np.einsum("bcxy,oc->boxy", win, K[:, :, kx, ky])
    return out


def col2im(dDhat: np.ndarray, b: int, c: int, n: int, k: int, s: int, p: int) -> np.ndarray:
    """Adjoint of ``lower``: scatter-add every lowered entry back to its source."""
    m = conv_out(n, k, s, p)
    g = dDhat.reshape(b, m, m, c, k, k).transpose(0, 3, 1, 2, 4, 5)  # b c x y kx ky
    padded = np.zeros((b, c, n + 2 * p, n + 2 * p))
    for kx in range(k):
        for ky in range(k):
            padded[:, :, kx:kx + s * (m - 1) + 1:s, ky:ky + s * (m - 1) + 1:s] += g[:, :, :, :, kx, ky]
    return padded[:, :, p:p + n, p:p + n]


# ------------------------------------------------------------- network ----
def layer_shapes(layers: list[dict], in_ch: int, in_size: int):
    """Walk a layer list (dicts; see paper_1606_04487_b200/nets.py) and return
    per-layer (input shape, output shape, param shapes).  Spatial shapes are
    (c, n, n); FC shapes are (features,)."""
    shapes = []
    cur = (in_ch, in_size, in_size)
    for L in layers:
        kind = L["kind"]
        params = []
        if kind == "conv":
            c, n, _ = cur
            m = conv_out(n, L["k"], L.get("stride", 1), L.get("pad", 0))
            params.append((L["d_out"], c, L["k"], L["k"]))
            if L.get("bias", True):
                params.append((L["d_out"],))
            out = (L["d_out"], m, m)
        elif kind == "pool":
            c, n, _ = cur
            o = pool_out(n, L["k"], L.get("stride", L["k"]), L.get("pad", 0), L.get("ceil", True))
            out = (c, o, o)
        elif kind == "relu":
            out = cur
        elif kind == "fc":
            f = int(np.prod(cur))
            params.append((f, L["d_out"]))
            if L.get("bias", True):
                params.append((L["d_out"],))
            out = (L["d_out"],)
        else:
            raise ValueError(f"unknown layer kind {kind!r}")
        shapes.append((cur, out, params))
        cur = out
    return shapes


def param_count(layers, in_ch, in_size) -> int:
    return sum(int(np.prod(p)) for _, _, ps in layer_shapes(layers, in_ch, in_size) for p in ps)


def unpack(layers, in_ch, in_size, W):
    """Flat W -> per-layer [weight, bias?] views, packed in layer order, weight
    before bias, C order (generalises problems.py:201-204)."""
    out, off = [], 0
    for _, _, params in layer_shapes(layers, in_ch, in_size):
        views = []
        for shp in params:
            sz = int(np.prod(shp))
            views.append(W[off:off + sz].reshape(shp))
            off += sz
        out.append(views)
    if off != W.size:
        raise ValueError(f"weight vector has {W.size} entries, net needs {off}")
    return out


def _pool_fwd(x, L):
    b, c, n, _ = x.shape
    k, s, p = L["k"], L.get("stride", L["k"]), L.get("pad", 0)
    o = pool_out(n, k, s, p, L.get("ceil", True))
    y = np.empty((b, c, o, o))
    arg = np.empty((b, c, o, o), dtype=np.int64) if L.get("mode", "max") == "max" else None
    for oy in range(o):
        for ox in range(o):
            hs, ws = oy * s - p, ox * s - p
            he, we = min(hs + k, n + p), min(ws + k, n + p)
            size = (he - hs) * (we - ws)
            hs, ws, he, we = max(hs, 0), max(ws, 0), min(he, n), min(we, n)
            win = x[:, :, hs:he, ws:we].reshape(b, c, -1)
            if arg is not None:
                j = np.argmax(win, axis=-1)  # first max in (dy, dx) order
                y[:, :, oy, ox] = np.take_along_axis(win, j[..., None], -1)[..., 0]
                wdt = we - ws
                arg[:, :, oy, ox] = (hs + j // wdt) * n + (ws + j % wdt)
            else:
                y[:, :, oy, ox] = win.sum(-1) / size
    return y, arg


def _pool_bwd(dy, x_shape, arg, L):
    b, c, n, _ = x_shape
    k, s, p = L["k"], L.get("stride", L["k"]), L.get("pad", 0)
    o = dy.shape[2]
    dx = np.zeros((b, c, n * n))
    if arg is not None:
        flat_arg = arg.reshape(b, c, -1)
        flat_dy = dy.reshape(b, c, -1)
        bi, ci = np.meshgrid(np.arange(b), np.arange(c), indexing="ij")
        for j in range(o * o):
            np.add.at(dx, (bi, ci, flat_arg[:, :, j]), flat_dy[:, :, j])
        return dx.reshape(b, c, n, n)
    dx = dx.reshape(b, c, n, n)
    for oy in range(o):
        for ox in range(o):
            hs, ws = oy * s - p, ox * s - p
            he, we = min(hs + k, n + p), min(ws + k, n + p)
            size = (he - hs) * (we - ws)
            hs, ws, he, we = max(hs, 0), max(ws, 0), min(he, n), min(we, n)
            dx[:, :, hs:he, ws:we] += (dy[:, :, oy, ox] / size)[:, :, None, None]
    return dx


def forward(layers, in_ch, in_size, W, X, workers: int = 1):
    """Returns (logits, cache).  X: (b, c, n, n) float64."""
    views = unpack(layers, in_ch, in_size, np.asarray(W, dtype=np.float64))
    h = np.asarray(X, dtype=np.float64)
    cache = []
    for L, (_, _, _), pv in zip(layers, layer_shapes(layers, in_ch, in_size), views):
        kind = L["kind"]
        if kind == "conv":
            s, p = L.get("stride", 1), L.get("pad", 0)
            z = conv_lowered(h, pv[0], s, p, workers=workers)
            if len(pv) > 1:
                z = z + pv[1][None, :, None, None]
            cache.append(("conv", h))
            h = z
        elif kind == "relu":
            cache.append(("relu", h))
            h = np.maximum(h, 0.0)
        elif kind == "pool":
            y, arg = _pool_fwd(h, L)
            cache.append(("pool", (h.shape, arg)))
            h = y
        elif kind == "fc":
            flat = h.reshape(h.shape[0], -1)
            z = flat @ pv[0]
            if len(pv) > 1:
                z = z + pv[1]
            cache.append(("fc", (h.shape, flat)))
            h = z
    return h, cache


def _partitions(b, workers):
    bounds = np.linspace(0, b, num=min(workers, b) + 1, dtype=int)
    return [(int(a), int(z)) for a, z in zip(bounds[:-1], bounds[1:]) if z > a]


def _par_rows(A, B, b, workers):
    """gemm(A, B) with A's rows split into contiguous image partitions, one
    thread each (the reference's conv_lowered partitioning, tensors.py:242-255)."""
    parts = _partitions(b, workers)
    rows = A.shape[0] // b
    out = np.empty((A.shape[0], B.shape[1]))

    def run(ab):
        lo, hi = ab
        out[lo * rows:hi * rows] = gemm(A[lo * rows:hi * rows], B)

    if len(parts) == 1:
        run(parts[0])
    else:
        with ThreadPoolExecutor(max_workers=len(parts)) as ex:
            list(ex.map(run, parts))
    return out


def _par_wgrad(Dhat, dR, b, workers):
    """Dhat^T dR summed over image partitions (fixed partition order)."""
    parts = _partitions(b, workers)
    rows = Dhat.shape[0] // b
    if len(parts) == 1:
        return gemm(Dhat.T, dR)
    with ThreadPoolExecutor(max_workers=len(parts)) as ex:
        partial = list(ex.map(lambda ab: gemm(Dhat[ab[0] * rows:ab[1] * rows].T,
                                              dR[ab[0] * rows:ab[1] * rows]), parts))
    out = partial[0]
    for q in partial[1:]:
        out = out + q
    return out


def softmax(logits):
    shifted = logits - logits.max(axis=1, keepdims=True)
    e = np.exp(shifted)
    return e / e.sum(axis=1, keepdims=True)


def xent(logits, y) -> float:
    """mean(lse - z_y) (problems.py:230-233)."""
    mx = logits.max(axis=1)
    lse = np.log(np.exp(logits - mx[:, None]).sum(axis=1)) + mx
    return float(np.mean(lse - logits[np.arange(len(y)), y]))


def loss(layers, in_ch, in_size, W, X, y, workers=1) -> float:
    return xent(forward(layers, in_ch, in_size, W, X, workers)[0], y)


def grad(layers, in_ch, in_size, W, X, y, workers: int = 1, return_acts: bool = False):
    """Mean-over-batch gradient in the flat W layout (problems.py:239-269)."""
    W = np.asarray(W, dtype=np.float64)
    logits, cache = forward(layers, in_ch, in_size, W, X, workers)
    views = unpack(layers, in_ch, in_size, W)
    b = logits.shape[0]
    pr = softmax(logits)
    pr[np.arange(b), y] -= 1.0
    dh = pr / b
    grads = [None] * len(layers)
    for li in range(len(layers) - 1, -1, -1):
        L, (kind, data), pv = layers[li], cache[li], views[li]
        if kind == "fc":
            in_shape, flat = data
            gw = flat.T @ dh
            gl = [gw] + ([dh.sum(axis=0)] if len(pv) > 1 else [])
            grads[li] = gl
            if li > 0:
                dh = (dh @ pv[0].T).reshape(in_shape)
        elif kind == "relu":
            dh = dh * (data > 0)
        elif kind == "pool":
            x_shape, arg = data
            dh = _pool_bwd(dh, x_shape, arg, L)
        elif kind == "conv":
            x = data
            s, p = L.get("stride", 1), L.get("pad", 0)
            b_, c, n, _ = x.shape
            d_out, _, k, _ = pv[0].shape
            m = conv_out(n, k, s, p)
            dR = dh.transpose(0, 2, 3, 1).reshape(b_ * m * m, d_out)
            Dhat = lower(x, k, s, p)
            gk = _par_wgrad(Dhat, dR, b_, workers).T.reshape(pv[0].shape)
            gl = [gk] + ([dR.sum(axis=0)] if len(pv) > 1 else [])
            grads[li] = gl
            if li > 0:
                dh = col2im(_par_rows(dR, lower_kernel(pv[0]).T, b_, workers), b_, c, n, k, s, p)
    flat = np.concatenate([g.ravel() for gl in grads if gl is not None for g in gl])
    if return_acts:
        return flat, logits
    return flat


# ------------------------------------------------- sgd.py restated ---------
def batch_stream(seed: int, group: int = 0) -> np.random.Generator:
    """PCG64(SeedSequence(seed, spawn_key=(1, group))) (sgd.py:28-35)."""
    return np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(1, group)))


def service_stream(seed: int, group: int) -> np.random.Generator:
    """(sgd.py:38-40)"""
    return np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(2, group)))


def problem_rng(seed: int, *key: int) -> np.random.Generator:
    """problems.py:19-20"""
    return np.random.default_rng(np.random.SeedSequence(seed, spawn_key=tuple(key)))


def sgd_step(W, V, g, w_read, eta, mu, lam):
    """V' = mu V - eta (g + lam w_read); W' = W + V' (sgd.py:92-101)."""
    V2 = mu * V - eta * (g + lam * w_read)
    return W + V2, V2


def tiny_cnn_data(image_size: int, classes: int, seed: int = 0, n_examples: int = 128):
    """The reference TinyCNN's synthetic data and teacher labels (problems.py:168-184)."""
    rng = problem_rng(seed, 0)
    images = rng.standard_normal((n_examples, 1, image_size, image_size))
    teacher = rng.standard_normal((classes, image_size * image_size))
    labels = np.argmax(teacher @ images.reshape(n_examples, -1).T, axis=0)
    return images, labels


def tiny_cnn_layers(image_size: int, classes: int):
    """conv 3x3 pad 1 1->4 (no bias) -> ReLU -> 2x2/2 max-pool -> linear (no bias)."""
    return [
        {"kind": "conv", "d_out": 4, "k": 3, "stride": 1, "pad": 1, "bias": False},
        {"kind": "relu"},
        {"kind": "pool", "mode": "max", "k": 2, "stride": 2, "pad": 0, "ceil": False},
        {"kind": "fc", "d_out": classes, "bias": False},
    ]


def run_sync(layers, in_ch, in_size, images, labels, W0, eta, mu, lam, b, steps, seed,
             sample_interval=1):
    """g = 1 loop (sgd.py:210-256) minus the stop rule: returns final W, V and
    the sampled full-dataset losses."""
    rng = batch_stream(seed)
    W = np.asarray(W0, dtype=np.float64).copy()
    V = np.zeros_like(W)
    losses = [loss(layers, in_ch, in_size, W, images, labels)]
    for t in range(1, steps + 1):
        idx = rng.integers(0, images.shape[0], size=b)
        g = grad(layers, in_ch, in_size, W, images[idx], labels[idx])
        W, V = sgd_step(W, V, g, W, eta, mu, lam)
        if t % sample_interval == 0 or t == steps:
            losses.append(loss(layers, in_ch, in_size, W, images, labels))
    return W, V, np.array(losses)


def simulate(grad_fn, sample_fn, W0, g, t_conv, t_fc, eta, mu, lam, b, max_updates, seed,
             exponential=False, models=None):
    """The g-group event loop (simulator.py:123-213) with a pluggable gradient.

    grad_fn(W, batch) -> gradient; sample_fn(rng, b) -> batch.  Returns
    (final W, final V, events) with events = [(group, read_step, write_step,
    staleness, start, enqueue, finish)].  ``models`` (a list) receives the
    master model after every write, initial model first (record_models).
    """
    brng = [batch_stream(seed, i) for i in range(g)]
    srng = [service_stream(seed, i) for i in range(g)] if exponential else None

    def services(i):
        if exponential:
            return srng[i].exponential(t_conv), srng[i].exponential(t_fc)
        return t_conv, t_fc

    W = np.asarray(W0, dtype=np.float64).copy()
    V = np.zeros_like(W)
    t = 0
    if models is not None:
        models.append(W.copy())
    heap, seq = [], 0
    for i in range(g):
        cd, fs = services(i)
        heapq.heappush(heap, (cd, seq, i, W.copy(), 0, 0.0, sample_fn(brng[i], b), fs))
        seq += 1
    fc_free = 0.0
    events = []
    while t < max_updates:
        conv_done, _, i, snap, read_step, read_time, batch, fs = heapq.heappop(heap)
        finish = max(fc_free, conv_done) + fs
        fc_free = finish
        W, V = sgd_step(W, V, grad_fn(snap, batch), snap, eta, mu, lam)
        t += 1
        events.append((i, read_step, t, t - 1 - read_step, read_time, conv_done, finish))
        if models is not None:
            models.append(W.copy())
        cd, fs2 = services(i)
        heapq.heappush(heap, (finish + cd, seq, i, W.copy(), t, finish, sample_fn(brng[i], b), fs2))
        seq += 1
    return W, V, events


def child_seed(seed: int, *key: int) -> int:
    """sgd.py:43-46"""
    return int(np.random.SeedSequence(seed, spawn_key=tuple(key)).generate_state(1, dtype=np.uint64)[0])


def estimate_implicit_momentum(grad_fn, full_grad_fn, sample_fn, W0, g, t_conv, t_fc, eta, lam, b,
                               max_updates, seed, n_runs, burn_in=None, signal_floor=0.02):
    """simulator.py:244-321 restated (exponential service, explicit mu = 0):
    average the master trajectories of runs seeded child_seed(seed, 3, r), then
    least-squares fit V(t+1) ~ a V(t) - c grad(W(t)) over the live-signal
    window; returns a.  (The reference also drops diverged runs; the oracle's
    callers use step sizes that do not diverge.)"""
    if burn_in is None:
        burn_in = 3 * g + 10
    paths = []
    for r in range(n_runs):
        models = []
        simulate(grad_fn, sample_fn, W0, g, t_conv, t_fc, eta, 0.0, lam, b, max_updates,
                 child_seed(seed, 3, r), exponential=True, models=models)
        paths.append(np.array(models))
    mean_path = np.mean(paths, axis=0)
    V = np.diff(mean_path, axis=0)
    mags = np.max(np.abs(V), axis=1)
    threshold = signal_floor * float(np.mean(mags[burn_in:burn_in + 10]))
    t_end = mean_path.shape[0] - 1
    for t in range(burn_in + 20, mean_path.shape[0] - 1):
        if mags[t] < threshold:
            t_end = t
            break
    X = np.concatenate([np.column_stack([V[t - 1], -full_grad_fn(mean_path[t])])
                        for t in range(burn_in + 1, t_end)])
    y = np.concatenate([V[t] for t in range(burn_in + 1, t_end)])
    beta, *_ = np.linalg.lstsq(X, y, rcond=None)
    return float(beta[0])


def deterministic_schedule(g: int, t: int):
    """Closed form of the deterministic g-group schedule for write step t >= 1:
    writer (t-1) mod g, read step max(0, t-g), staleness min(t-1, g-1), batch
    draw floor((t-1)/g) of the writer's stream."""
    return (t - 1) % g, max(0, t - g), min(t - 1, g - 1), (t - 1) // g


def cpu_count() -> int:
    return os.cpu_count() or 1
