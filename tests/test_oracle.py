"""Pin the CPU oracle (oracle/refcnn.py) before trusting it.

(1) Against fixtures produced by running the reference itself
    (tests/golden/make_golden.py): lowering bit-exact, conv/gemm/lift, the
    TinyCNN loss and gradient, run_sync weights, the g-group simulator's event
    schedule and weights, and the SPEC KATs.
(2) The restated extensions (bias, overlapping/average/ceil pooling, FC
    stacks, conv input gradient) against central finite differences and the
    lowering/col2im adjoint identity.
"""

import os

import numpy as np
import pytest

from oracle import refcnn as R

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name))


def test_lower_bit_exact_vs_reference():
    z = load("lower.npz")
    i = 0
    while f"case{i}_geom" in z:
        b, c, n, k, s, p, start, b_p = z[f"case{i}_geom"]
        got = R.lower(z[f"case{i}_D"], int(k), int(s), int(p), int(start), int(b_p))
        assert np.array_equal(got, z[f"case{i}_Dhat"]), i
        i += 1
    assert i >= 5


def test_conv_gemm_lift_vs_reference():
    z = load("conv.npz")
    i = 0
    while f"conv{i}_geom" in z:
        n, k, din, dout, s, p, b = (int(v) for v in z[f"conv{i}_geom"])
        D, K = z[f"conv{i}_D"], z[f"conv{i}_K"]
        for workers, b_p in ((1, b), (2, 1), (3, 2)):
            got = R.conv_lowered(D, K, s, p, b_p=b_p, workers=workers)
            np.testing.assert_allclose(got, z[f"conv{i}_R"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(R.conv_direct(D, K, s, p), z[f"conv{i}_Rdirect"], rtol=0, atol=1e-12)
        i += 1
    assert np.array_equal(R.conv_lowered(z["kat_D"], z["kat_K"]), z["kat_R"])
    assert np.array_equal(z["kat_R"].reshape(2, 2), np.array([[6.0, 8.0], [12.0, 14.0]]))
    np.testing.assert_allclose(R.gemm(z["gemm_A"], z["gemm_B"]), z["gemm_C"], rtol=0, atol=1e-12)
    assert np.array_equal(z["gemm_kat"], np.array([[17.0], [39.0]]))


@pytest.mark.parametrize("tag", ["s8c4", "s16c10"])
def test_tiny_cnn_vs_reference(tag):
    z = load("tinycnn.npz")
    size, classes, n_ex, b, seed = (int(v) for v in z[f"{tag}_meta"])
    images, labels = R.tiny_cnn_data(size, classes, seed, n_ex)
    assert np.array_equal(images, z[f"{tag}_images"]) and np.array_equal(labels, z[f"{tag}_labels"])
    W0 = 0.01 * R.problem_rng(seed, 1).standard_normal(R.param_count(R.tiny_cnn_layers(size, classes), 1, size))
    assert np.array_equal(W0, z[f"{tag}_W0"])
    idx = R.batch_stream(seed).integers(0, n_ex, size=b)
    assert np.array_equal(images[idx], z[f"{tag}_bx"])
    layers = R.tiny_cnn_layers(size, classes)
    g = R.grad(layers, 1, size, W0, z[f"{tag}_bx"], z[f"{tag}_by"])
    np.testing.assert_allclose(g, z[f"{tag}_grad"], rtol=0, atol=1e-14)
    assert abs(R.loss(layers, 1, size, W0, z[f"{tag}_bx"], z[f"{tag}_by"]) - float(z[f"{tag}_loss"])) < 1e-13
    assert abs(R.loss(layers, 1, size, W0, images, labels) - float(z[f"{tag}_full_loss"])) < 1e-13


def test_run_sync_vs_reference():
    z = load("tinycnn.npz")
    eta, mu, lam, b, steps, seed = z["sync_hp"]
    images, labels = R.tiny_cnn_data(8, 4, 3, 64)
    layers = R.tiny_cnn_layers(8, 4)
    W0 = 0.01 * R.problem_rng(3, 1).standard_normal(R.param_count(layers, 1, 8))
    W, V, losses = R.run_sync(layers, 1, 8, images, labels, W0, eta, mu, lam, int(b), int(steps), int(seed))
    np.testing.assert_allclose(W, z["sync_W"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(V, z["sync_V"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(losses, z["sync_losses"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("mode", ["deterministic", "exponential"])
def test_simulate_schedule_vs_reference(mode):
    z = load("tinycnn.npz")
    images, labels = R.tiny_cnn_data(8, 4, 3, 64)
    layers = R.tiny_cnn_layers(8, 4)
    W0 = 0.01 * R.problem_rng(3, 1).standard_normal(R.param_count(layers, 1, 8))

    def grad_fn(W, batch):
        return R.grad(layers, 1, 8, W, *batch)

    def sample_fn(rng, b):
        idx = rng.integers(0, 64, size=b)
        return images[idx], labels[idx]

    # T_cc=8, T_nc=0.1, t_fc=0.5; t_conv(k) = max(T_cc/k, T_nc*k) (cluster.py:76-80)
    if mode == "deterministic":
        g, k, ev, Wk, n, seed = 4, 2, "sim_events", "sim_W", 12, 5
    else:
        g, k, ev, Wk, n, seed = 8, 1, "simexp_events", "simexp_W", 20, 7
    t_conv = max(8.0 / k, 0.1 * k)
    W, V, events = R.simulate(grad_fn, sample_fn, W0, g, t_conv, 0.5, 0.05, 0.9, 1e-3, 16, n, seed,
                              exponential=(mode == "exponential"))
    got = np.array(events)
    np.testing.assert_array_equal(got[:, :4], z[ev][:, :4])
    np.testing.assert_allclose(got[:, 4:], z[ev][:, 4:], rtol=0, atol=1e-12)
    np.testing.assert_allclose(W, z[Wk], rtol=0, atol=1e-13)
    if mode == "deterministic":
        for t in range(1, n + 1):
            writer, read, stale, _ = R.deterministic_schedule(g, t)
            row = got[t - 1]
            assert (row[0], row[1], row[3]) == (writer, read, stale)


def test_sgd_kat():
    z = load("tinycnn.npz")
    W, V = R.sgd_step(np.array([1.0]), np.array([0.0]), np.array([2.0]), np.array([1.0]), 0.1, 0.9, 0.0)
    assert np.allclose([W[0], V[0]], z["sgd_kat"]) and np.allclose([W[0], V[0]], [0.8, -0.2])


# ---------------------------------------------------- extensions, pinned --
SMALL_NET = [
    {"kind": "conv", "d_out": 3, "k": 3, "stride": 1, "pad": 1, "bias": True},
    {"kind": "relu"},
    {"kind": "pool", "mode": "max", "k": 3, "stride": 2, "pad": 0, "ceil": True},
    {"kind": "conv", "d_out": 4, "k": 3, "stride": 2, "pad": 1, "bias": True},
    {"kind": "relu"},
    {"kind": "pool", "mode": "avg", "k": 3, "stride": 2, "pad": 0, "ceil": True},
    {"kind": "fc", "d_out": 5, "bias": True},
    {"kind": "relu"},
    {"kind": "fc", "d_out": 3, "bias": True},
]


def test_extensions_finite_differences():
    rng = np.random.default_rng(0)
    in_ch, size, b = 2, 11, 3
    dim = R.param_count(SMALL_NET, in_ch, size)
    W = 0.5 * rng.standard_normal(dim)
    X = rng.standard_normal((b, in_ch, size, size))
    y = rng.integers(0, 3, size=b)
    g = R.grad(SMALL_NET, in_ch, size, W, X, y)
    eps = 1e-6
    for j in rng.choice(dim, size=40, replace=False):
        e = np.zeros(dim)
        e[j] = eps
        fd = (R.loss(SMALL_NET, in_ch, size, W + e, X, y) - R.loss(SMALL_NET, in_ch, size, W - e, X, y)) / (2 * eps)
        assert abs(fd - g[j]) <= 1e-6 + 1e-4 * abs(fd), (j, fd, g[j])


@pytest.mark.parametrize("geom", [(2, 3, 9, 3, 1, 1), (1, 2, 13, 5, 2, 2), (2, 3, 27, 11, 4, 0)])
def test_col2im_adjoint(geom):
    b, c, n, k, s, p = geom
    rng = np.random.default_rng(1)
    D = rng.standard_normal((b, c, n, n))
    m = R.conv_out(n, k, s, p)
    G = rng.standard_normal((b * m * m, c * k * k))
    lhs = float((R.lower(D, k, s, p) * G).sum())
    rhs = float((D * R.col2im(G, b, c, n, k, s, p)).sum())
    assert abs(lhs - rhs) <= 1e-10 * max(1.0, abs(lhs))


def test_pool_geometry_caffe_rule():
    assert R.pool_out(32, 3, 2, 0, True) == 16   # CIFAR-10 quick pool1
    assert R.pool_out(32, 3, 2, 0, False) == 15
    assert R.pool_out(55, 3, 2, 0, True) == 27   # CaffeNet pool1
    assert R.pool_out(13, 3, 2, 0, True) == 6    # CaffeNet pool5
    assert R.pool_out(24, 2, 2, 0, True) == 12   # LeNet pool1
    assert R.pool_out(7, 3, 2, 1, True) == 4


def test_conv_geometry_errors_match_reference_rules():
    with pytest.raises(ValueError):
        R.conv_out(5, 7, 1, 0)
    with pytest.raises(ValueError):
        R.conv_out(8, 3, 2, 0)


def test_implicit_momentum_estimator_vs_reference():
    """oracle restatement of simulator.py:244-321 == the reference's estimator."""
    z = load("implicit_momentum.npz")
    size, classes, n_ex, pseed, eta, b, T_cc, t_fc, max_updates, seed, n_runs = z["im_cfg"]
    size, classes, n_ex, b = int(size), int(classes), int(n_ex), int(b)
    images, labels = R.tiny_cnn_data(size, classes, int(pseed), n_ex)
    layers = R.tiny_cnn_layers(size, classes)
    W0 = 0.01 * R.problem_rng(int(pseed), 1).standard_normal(R.param_count(layers, 1, size))

    def grad_fn(W, batch):
        return R.grad(layers, 1, size, W, *batch)

    def full_grad_fn(W):
        return R.grad(layers, 1, size, W, images, labels)

    def sample_fn(rng, bb):
        idx = rng.integers(0, n_ex, size=bb)
        return images[idx], labels[idx]

    for g in (2, 4):   # N = 4, T_nc = 0: t_conv(k) = T_cc / k (cluster.py:76-80)
        a = R.estimate_implicit_momentum(grad_fn, full_grad_fn, sample_fn, W0, g, T_cc / (4 // g),
                                         t_fc, eta, 0.0, b, int(max_updates), int(seed), int(n_runs))
        assert abs(a - float(z[f"im_g{g}"])) < 1e-9, (g, a, float(z[f"im_g{g}"]))
