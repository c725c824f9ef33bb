"""Free-running asynchronous groups (async_groups.py) on CPU with gloo.

The arrival order is not reproducible (random compute delays), so parity is
against the run's own update log: the log must describe a valid asynchronous
schedule (each group reads the model right after its own previous write,
FIFO write steps 1..T, staleness = write - 1 - read), and replaying it in
order must reproduce the server's final model bit for bit."""

import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import dist_worker as DW

HP = (0.05, 0.0, 1e-3, 16)


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,g", [(3, 2), (3, 1), (5, 2)])
def test_async_log_is_a_valid_schedule_and_replays_exactly(world, g, tmp_path):
    T = 12
    mp.spawn(DW.async_worker, args=(world, free_port(), g, T, HP, str(tmp_path)), nprocs=world,
             join=True)
    ev = np.load(tmp_path / "ev.npy")
    W, Wr = np.load(tmp_path / "W.npy"), np.load(tmp_path / "Wreplay.npy")
    assert ev.shape[0] == T and np.array_equal(ev[:, 2], np.arange(1, T + 1))
    assert np.array_equal(ev[:, 3], ev[:, 2] - 1 - ev[:, 1]) and (ev[:, 3] >= 0).all()
    for i in range(g):
        mine = ev[ev[:, 0] == i]
        assert np.array_equal(mine[:, 4], np.arange(len(mine)))          # j-th draw of its stream
        assert mine[0, 1] == 0
        assert np.array_equal(mine[1:, 1], mine[:-1, 2])                 # reads right after its write
    assert set(ev[:, 0].tolist()) == set(range(g))
    assert np.array_equal(W, Wr)


@pytest.mark.parametrize("world,g", [(2, 2), (2, 1), (4, 2), (4, 4)])
def test_colocated_server_log_is_valid_and_replays(world, g, tmp_path):
    """The co-located runtime (server thread on rank 0, no extra process):
    N ranks map g groups of k = N/g (cluster.py:54-73); the log is a valid
    asynchronous schedule and replays to the server's final model (exactly for
    k <= 2, where the group sum a + b is order-independent)."""
    T = 12
    mp.spawn(DW.colocated_worker, args=(world, free_port(), g, T, HP, str(tmp_path)), nprocs=world,
             join=True)
    ev = np.load(tmp_path / "ev.npy")
    W, Wr = np.load(tmp_path / "W.npy"), np.load(tmp_path / "Wreplay.npy")
    assert ev.shape[0] == T and np.array_equal(ev[:, 2], np.arange(1, T + 1))
    assert np.array_equal(ev[:, 3], ev[:, 2] - 1 - ev[:, 1]) and (ev[:, 3] >= 0).all()
    for i in range(g):
        mine = ev[ev[:, 0] == i]
        assert len(mine) > 0 and mine[0, 1] == 0
        assert np.array_equal(mine[:, 4], np.arange(len(mine)))
        assert np.array_equal(mine[1:, 1], mine[:-1, 2])
    if world // g <= 2:
        assert np.array_equal(W, Wr)
    else:
        assert np.allclose(W, Wr, rtol=0, atol=1e-12)
