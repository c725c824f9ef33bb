"""Worker for the multi-process (gloo, CPU) tests of groups.GroupRuntime.

The runtime's collective/schedule logic runs unchanged; gradients and updates
come from the float64 CPU oracle (a test double for the CUDA backend)."""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle import refcnn as R  # noqa: E402
from paper_1606_04487_b200.cluster import ExecutionPlan  # noqa: E402
from paper_1606_04487_b200.groups import GroupRuntime  # noqa: E402
from paper_1606_04487_b200.sgd import Hyperparams  # noqa: E402

SIZE, CLASSES, N_EX, SEED = 8, 4, 64, 3


class OracleBackend:
    device = torch.device("cpu")

    def __init__(self):
        self.layers = R.tiny_cnn_layers(SIZE, CLASSES)
        self.images, self.labels = R.tiny_cnn_data(SIZE, CLASSES, SEED, N_EX)

    def grad(self, W, idx):
        g = R.grad(self.layers, 1, SIZE, W.numpy(), self.images[idx], self.labels[idx])
        return torch.from_numpy(g)

    def sgd(self, W, V, G, w_read, hp):
        V.mul_(hp.mu).sub_(hp.eta * (G + hp.lam * w_read))
        W.add_(V)


def initial_weights():
    layers = R.tiny_cnn_layers(SIZE, CLASSES)
    return 0.01 * R.problem_rng(SEED, 1).standard_normal(R.param_count(layers, 1, SIZE))


def worker(rank, world, port, g, rounds, hp_tuple, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        eta, mu, lam, b = hp_tuple
        hp = Hyperparams(eta=eta, mu=mu, lam=lam, b=b)
        rt = GroupRuntime(ExecutionPlan(world, g), OracleBackend(), hp,
                          torch.from_numpy(initial_weights()), N_EX, seed=11)
        rt.run(rounds)
        np.save(os.path.join(out_dir, f"W{rank}.npy"), rt.W.numpy())
        np.save(os.path.join(out_dir, f"ev{rank}.npy"),
                np.array([[e.group_id, e.read_step, e.write_step, e.staleness] for e in rt.events]))
    finally:
        dist.destroy_process_group()
