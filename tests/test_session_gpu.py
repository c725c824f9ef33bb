"""DeviceSession execution modes must not change the math: eager steps, CUDA
graph replay, and host batches prefetched on a copy stream give bit-identical
weights for the same batches."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_1606_04487_b200 as P  # noqa: E402
from paper_1606_04487_b200.problems import CNNProblem, DeviceBatch, HostBatch  # noqa: E402


@pytest.mark.parametrize("net,b", [("lenet", 16), ("cifar10_quick", 8)])
def test_graph_replay_equals_eager(net, b):
    prob = CNNProblem(net, n_examples=64, seed=2, precision="tf32")
    hp = P.Hyperparams(eta=0.01, mu=0.9, lam=5e-4, b=b)
    rng = np.random.default_rng(0)
    batches = [torch.from_numpy(rng.integers(0, 64, size=b)).cuda() for _ in range(6)]
    state = prob.initial_state()
    out = []
    for use_graph in (False, True):
        sess = prob.device_session(state, hp)
        sess.use_graph = use_graph and sess.use_graph   # OMNI_NO_GRAPH wins
        losses = []
        for i, idx in enumerate(batches):
            sess.step(DeviceBatch(idx))
            try:
                losses.append(sess.last_loss())
            except RuntimeError as e:   # name the failing step for triage
                raise RuntimeError(f"{net}: use_graph={sess.use_graph} step={i} "
                                   f"graphs={list(sess._graphs)}") from e
        assert bool(sess._graphs) == sess.use_graph
        out.append((sess.W.clone(), sess.V.clone(), losses, sess.t))
    (W0, V0, l0, t0), (W1, V1, l1, t1) = out
    assert t0 == t1 == 6
    assert torch.equal(W0, W1) and torch.equal(V0, V1) and l0 == l1


@pytest.mark.parametrize("net,b", [("cifar10_quick", 8), ("caffenet", 4)])
def test_prefetched_host_batches_equal_device_batches(net, b):
    """caffenet: the host batch goes through the zero-copy space-to-depth kernel
    (transfer + conv1 layout in one pass); the device batch through the fused
    gather + space-to-depth.  Both must give the same weights, bit for bit."""
    prob = CNNProblem(net, n_examples=32, seed=5, precision="tf32")
    hp = P.Hyperparams(eta=0.01, mu=0.9, b=b)
    state = prob.initial_state()
    rng = np.random.default_rng(1)
    idxs = [rng.integers(0, 32, size=b) for _ in range(6)]
    a = prob.device_session(state, hp, use_graph=False)
    for idx in idxs:
        a.step(DeviceBatch(torch.from_numpy(idx).cuda()))
    sb = prob.device_session(state, hp)   # graphed: steps 2.. replay per-slot graphs
    hbs = [HostBatch(prob.data[torch.from_numpy(i).cuda()].cpu().pin_memory(),
                     prob.data_labels[torch.from_numpy(i).cuda()].cpu().pin_memory()) for i in idxs]
    sb.prefetch(hbs[0])
    for i, hb in enumerate(hbs):
        sb.step(hb)
        if i + 1 < len(hbs):
            sb.prefetch(hbs[i + 1])
    torch.cuda.synchronize()
    assert torch.equal(a.W, sb.W) and torch.equal(a.V, sb.V)


def test_loss_future_matches_last_loss():
    prob = CNNProblem("lenet", n_examples=32, seed=3, precision="tf32")
    hp = P.Hyperparams(eta=0.01, mu=0.9, b=8)
    sess = prob.device_session(prob.initial_state(), hp)
    futs, sync = [], []
    for i in range(5):
        sess.step(DeviceBatch(torch.arange(i, i + 8).cuda()))
        futs.append(sess.loss_future())
        if i >= 2:   # results read lagging behind, like bench.py's e2e loop
            futs[i - 2].result()
        sync.append(sess.last_loss())
    assert [f.result() for f in futs] == sync


def test_ragged_batch_step_equals_oracle_update():
    """A step on a batch smaller than the session's b (the eager path) is the
    momentum update with the mean gradient over exactly those images."""
    from oracle import refcnn as R

    prob = CNNProblem("lenet", n_examples=32, seed=6, precision="3xtf32")
    hp = P.Hyperparams(eta=0.05, mu=0.9, lam=1e-3, b=8)
    state = prob.initial_state()
    sess = prob.device_session(state, hp)
    idx = np.array([3, 17, 5, 29, 11])                       # 5 < b = 8
    sess.step(DeviceBatch(torch.from_numpy(idx).cuda()))
    X = prob.data[torch.from_numpy(idx).cuda()].permute(0, 3, 1, 2).double().cpu().numpy()
    y = prob.data_labels[torch.from_numpy(idx).cuda()].long().cpu().numpy()
    g = R.grad(prob.net.to_dicts(), 1, 28, state.W, X, y)
    V = -hp.eta * (g + hp.lam * state.W)
    W = state.W + V
    got = sess.W.double().cpu().numpy()
    assert np.linalg.norm(got - W) / np.linalg.norm(W) < 1e-6


def test_empty_batch_fails_loudly():
    prob = CNNProblem("lenet", n_examples=16, seed=6, precision="tf32")
    sess = prob.device_session(prob.initial_state(), P.Hyperparams(eta=0.01, b=8))
    with pytest.raises((ValueError, RuntimeError)):
        sess.step(DeviceBatch(torch.zeros(0, dtype=torch.int64, device="cuda")))


def test_prefetch_refuses_a_third_outstanding_batch():
    """Two staging slots: a third prefetch before any of the two staged batches
    is stepped must fail loudly instead of overwriting a staged slot."""
    prob = CNNProblem("lenet", n_examples=32, seed=3, precision="tf32")
    sess = prob.device_session(prob.initial_state(), P.Hyperparams(eta=0.01, mu=0.9, b=8))
    hbs = [HostBatch(torch.randn(8, 28, 28, 1).pin_memory(),
                     torch.randint(0, 10, (8,), dtype=torch.int32).pin_memory()) for _ in range(4)]
    sess.prefetch(hbs[0])
    sess.prefetch(hbs[1])
    with pytest.raises(ValueError, match="staging slots"):
        sess.prefetch(hbs[2])
    sess.step(hbs[0])                   # frees slot 0
    sess.prefetch(hbs[2])
    sess.step(hbs[1])
    sess.step(hbs[2])
    sess.step(hbs[3])                   # never prefetched: plain upload path
    assert np.isfinite(sess.last_loss())
