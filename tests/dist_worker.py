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

    def group_updates(self, rows, members, W, V, snaps, hp):
        for i, ms in enumerate(members):
            Gi = rows[ms[0]].clone()[:W.numel()]
            for m in ms[1:]:
                Gi.add_(rows[m][:W.numel()])
            self.sgd(W, V, Gi, snaps[i], hp)
            snaps[i].copy_(W)

    def exchange(self, plan):
        return TorchExchange(plan)


class TorchExchange:
    """groups.GroupRuntime's collectives over torch.distributed (gloo): the
    CPU test double of comm.GroupExchange, method for method."""

    def __init__(self, plan):
        self.plan = plan
        self.rank = dist.get_rank()
        # every rank creates every subgroup, in the same order
        self.groups = [dist.new_group(plan.group_ranks(i)) for i in range(plan.g)]
        self.crosses = [dist.new_group([i * plan.k + j for i in range(plan.g)]) for j in range(plan.k)]

    def group_allreduce(self, t):
        dist.all_reduce(t, group=self.groups[self.plan.group_of(self.rank)])

    def cross_allgather(self, t, out):
        dist.all_gather(list(out.view(self.plan.g, -1)), t,
                        group=self.crosses[self.plan.member_of(self.rank)])

    def world_allreduce(self, t):
        dist.all_reduce(t)

    def world_allgather(self, t, out):
        dist.all_gather(list(out.view(self.plan.N, -1)), t)

    def all_to_all(self, parts, recv):
        dist.all_to_all_single(recv, torch.cat(parts))

    def all_to_all_async(self, parts, recv):
        return dist.all_to_all_single(recv, torch.cat(parts), async_op=True)


def initial_weights():
    layers = R.tiny_cnn_layers(SIZE, CLASSES)
    return 0.01 * R.problem_rng(SEED, 1).standard_normal(R.param_count(layers, 1, SIZE))


def worker(rank, world, port, g, rounds, hp_tuple, out_dir, sharded=True):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        eta, mu, lam, b = hp_tuple
        hp = Hyperparams(eta=eta, mu=mu, lam=lam, b=b)
        rt = GroupRuntime(ExecutionPlan(world, g), OracleBackend(), hp,
                          torch.from_numpy(initial_weights()), N_EX, seed=11, sharded=sharded)
        rt.run(rounds)
        np.save(os.path.join(out_dir, f"W{rank}.npy"), rt.W.numpy())
        np.save(os.path.join(out_dir, f"ev{rank}.npy"),
                np.array([[e.group_id, e.read_step, e.write_step, e.staleness] for e in rt.events]))
    finally:
        dist.destroy_process_group()


class JitterBackend(OracleBackend):
    """OracleBackend with random compute delays: the asynchronous arrival order
    then differs from run to run (what replay must be robust to)."""

    def __init__(self, seed):
        super().__init__()
        self.rng = np.random.default_rng(seed)

    def grad(self, W, idx):
        import time

        time.sleep(float(self.rng.uniform(0.0, 0.02)))
        return super().grad(W, idx)


def async_worker(rank, world, port, g, max_updates, hp_tuple, out_dir):
    """paper_1606_04487_b200.async_groups: rank 0 serves, ranks 1.. compute."""
    from paper_1606_04487_b200 import async_groups as A

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        eta, mu, lam, b = hp_tuple
        hp = Hyperparams(eta=eta, mu=mu, lam=lam, b=b)
        plan = ExecutionPlan(world - 1, g)
        W0 = torch.from_numpy(initial_weights())
        if rank == 0:
            res = A.run_server(plan, OracleBackend(), hp, W0, max_updates)
            Wr, _ = A.replay(res.events, plan, OracleBackend(), hp, W0, N_EX, seed=11)
            np.save(os.path.join(out_dir, "W.npy"), res.W.numpy())
            np.save(os.path.join(out_dir, "Wreplay.npy"), Wr.numpy())
            np.save(os.path.join(out_dir, "ev.npy"),
                    np.array([[e.group_id, e.read_step, e.write_step, e.staleness, e.batch_index]
                              for e in res.events]))
        else:
            A.run_worker(plan, JitterBackend(1000 + rank), hp, W0, N_EX, seed=11)
    finally:
        dist.destroy_process_group()


def colocated_worker(rank, world, port, g, max_updates, hp_tuple, out_dir):
    """paper_1606_04487_b200.colocated: every rank computes, rank 0 also serves
    (host shared-memory payload store, gloo group collectives)."""
    from paper_1606_04487_b200 import async_groups as A
    from paper_1606_04487_b200 import colocated as C

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        eta, mu, lam, b = hp_tuple
        hp = Hyperparams(eta=eta, mu=mu, lam=lam, b=b)
        plan = ExecutionPlan(world, g)
        W0 = torch.from_numpy(initial_weights())
        res = C.run_colocated(plan, JitterBackend(1000 + rank), hp, W0, N_EX, seed=11,
                              max_updates=max_updates, store="shm")
        if rank == 0:
            Wr, _ = A.replay(res.events, plan, OracleBackend(), hp, W0, N_EX, seed=11)
            np.save(os.path.join(out_dir, "W.npy"), res.W.numpy())
            np.save(os.path.join(out_dir, "Wreplay.npy"), Wr.numpy())
            np.save(os.path.join(out_dir, "ev.npy"),
                    np.array([[e.group_id, e.read_step, e.write_step, e.staleness, e.batch_index]
                              for e in res.events]))
    finally:
        dist.destroy_process_group()
