"""N > 1 compute-group runtime on CPU with gloo (world sizes 2 and 4).

GroupRuntime's schedule and collectives must reproduce, in float64, the
reference's single-process semantics: g = 1 with k ranks == run_sync with the
group batch (sgd.py:210-256); g > 1 == simulate(service_mode="deterministic")
(simulator.py:123-213), event log and weights."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import dist_worker as DW
from oracle import refcnn as R

HP = (0.05, 0.9, 1e-3, 16)


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run(world, g, rounds, tmp_path, sharded=True):
    mp.spawn(DW.worker, args=(world, free_port(), g, rounds, HP, str(tmp_path), sharded), nprocs=world,
             join=True)
    Ws = [np.load(tmp_path / f"W{r}.npy") for r in range(world)]
    evs = [np.load(tmp_path / f"ev{r}.npy") for r in range(world)]
    for r in range(1, world):   # every rank holds the same master model and log
        assert np.array_equal(Ws[r], Ws[0]) and np.array_equal(evs[r], evs[0])
    return Ws[0], evs[0]


def oracle_simulate(g, updates):
    layers = R.tiny_cnn_layers(DW.SIZE, DW.CLASSES)
    images, labels = R.tiny_cnn_data(DW.SIZE, DW.CLASSES, DW.SEED, DW.N_EX)

    def grad_fn(W, batch):
        return R.grad(layers, 1, DW.SIZE, W, *batch)

    def sample_fn(rng, b):
        idx = rng.integers(0, DW.N_EX, size=b)
        return images[idx], labels[idx]

    eta, mu, lam, b = HP
    W, V, ev = R.simulate(grad_fn, sample_fn, DW.initial_weights(), g, 4.0, 0.5, eta, mu, lam, b,
                          updates, seed=11)
    return W, np.array([e[:4] for e in ev])


def nrel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_g1_k2_equals_run_sync(tmp_path):
    W, ev = run(2, 1, 5, tmp_path)
    layers = R.tiny_cnn_layers(DW.SIZE, DW.CLASSES)
    images, labels = R.tiny_cnn_data(DW.SIZE, DW.CLASSES, DW.SEED, DW.N_EX)
    eta, mu, lam, b = HP
    Wr, _, _ = R.run_sync(layers, 1, DW.SIZE, images, labels, DW.initial_weights(), eta, mu, lam, b, 5, 11)
    assert nrel(W, Wr) < 1e-12
    assert np.array_equal(ev[:, 3], np.zeros(5))   # synchronous: staleness 0


def test_g2_k1_equals_deterministic_simulate(tmp_path):
    W, ev = run(2, 2, 4, tmp_path)
    Wr, evr = oracle_simulate(2, 8)
    assert np.array_equal(ev, evr)
    assert nrel(W, Wr) < 1e-12


def test_g2_k1_replicated_equals_deterministic_simulate(tmp_path):
    # sharded=False: every rank holds W, V and all g snapshots; group allreduce
    # + cross-group all-gather + the g ordered updates in one group_updates call
    W, ev = run(2, 2, 4, tmp_path, sharded=False)
    Wr, evr = oracle_simulate(2, 8)
    assert np.array_equal(ev, evr)
    assert nrel(W, Wr) < 1e-12


@pytest.mark.slow
def test_g2_k2_world4(tmp_path):
    W, ev = run(4, 2, 3, tmp_path)
    Wr, evr = oracle_simulate(2, 6)
    assert np.array_equal(ev, evr)
    assert nrel(W, Wr) < 1e-12
