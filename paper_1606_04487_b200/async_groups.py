"""Free-running asynchronous compute groups on real GPUs.

The reference models asynchrony as a discrete-event simulation
(simulator.py:123-213): g groups snapshot the master model, compute a
gradient for t_conv(k), and a single serial server applies the updates FIFO,
each with the gradient evaluated at the group's snapshot (stale_step,
sgd.py:104-112).  Here the same protocol runs for real, one process per GPU:

* rank 0 is the server: it holds the master W, V in HBM, keeps one posted
  receive per group leader, and applies each gradient as soon as it has
  arrived (FIFO in order of arrival), then sends that group a fresh
  snapshot (preceded by a continue/stop flag);
* ranks 1..N are workers in g groups of k = N/g; a group computes its
  gradient data parallel (allreduce inside the group), its leader pushes it
  to the server and receives the next snapshot, which it broadcasts to the
  group.  No group ever waits for another group.

Every applied update is logged as (group, read_step, write_step, staleness,
time); ``replay`` re-applies that log deterministically, which reproduces the
asynchronous run's final model exactly (same kernels, same batches) -- the
parity check for a schedule that is not reproducible by construction.  The
log feeds staleness_stats / measured_he and the HE model comparison
(cluster.he_predict).

The gradient/update provider is pluggable (``groups.Backend``): the B200
engine in production, a CPU backend in the gloo tests.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .cluster import ExecutionPlan
from .sgd import Hyperparams, batch_stream


@dataclass(frozen=True)
class AsyncEvent:
    group_id: int
    read_step: int
    write_step: int
    staleness: int
    arrive_time: float   # server clock (s since start) when the update was applied
    batch_index: int     # j-th gradient of this group (its j-th draw from its batch stream)


@dataclass
class AsyncResult:
    events: list
    W: torch.Tensor
    V: torch.Tensor
    seconds: float

    @property
    def write_times(self) -> np.ndarray:
        return np.array([e.arrive_time for e in self.events])


def worker_ranks(plan: ExecutionPlan, group: int) -> list[int]:
    """Global ranks of a group's workers (rank 0 is the server)."""
    return [1 + group * plan.k + j for j in range(plan.k)]


def _new_groups(plan: ExecutionPlan):
    """Intra-group process groups, plus (NCCL) one server<->leader group per
    worker group: point-to-point traffic of different groups then runs on
    separate communicators / streams, so a receive still pending from one
    group never queues the replies to another (on one shared P2P stream the
    groups end up taking turns).  Every rank creates every subgroup, in the
    same order (torch.distributed rule)."""
    intra = [dist.new_group(worker_ranks(plan, i)) for i in range(plan.g)]
    if dist.get_backend() == "nccl":
        pair = [dist.new_group([0, worker_ranks(plan, i)[0]]) for i in range(plan.g)]
    else:   # gloo: the server's any-source receive needs the default group
        pair = [None] * plan.g
    return intra, pair


def run_server(plan: ExecutionPlan, backend, hp: Hyperparams, W0: torch.Tensor,
               max_updates: int) -> AsyncResult:
    """Rank 0.  Returns the update log and the final master model."""
    if dist.get_rank() != 0:
        raise RuntimeError("run_server runs on rank 0")
    _, pair = _new_groups(plan)
    dev = W0.device
    W = W0.clone()
    V = torch.zeros_like(W)
    hp_sum = hp.replace(eta=hp.eta / plan.k, lam=hp.lam * plan.k)   # groups send sums of k means
    leaders = [worker_ranks(plan, i)[0] for i in range(plan.g)]
    bufs = [torch.empty_like(W) for _ in range(plan.g)]
    snaps = [W0.clone() for _ in range(plan.g)]   # what each group currently computes on
    read_step = [0] * plan.g
    drawn = [0] * plan.g
    go = torch.ones(1, dtype=torch.int32, device=dev)
    stop = torch.zeros(1, dtype=torch.int32, device=dev)
    events: list[AsyncEvent] = []
    # Arrival detection: NCCL -- one posted receive per group leader, polled
    # (Work.is_completed queries the receive's CUDA event); gloo -- a blocking
    # any-source receive (its Work objects only complete inside wait()).
    nccl = dist.get_backend() == "nccl"
    by_leader = {r: i for i, r in enumerate(leaders)}
    anybuf = None if nccl else torch.empty_like(W)
    pending = ([dist.irecv(bufs[i], src=leaders[i], group=pair[i]) for i in range(plan.g)]
               if nccl else None)

    def next_arrival() -> int:
        if not nccl:
            src = dist.recv(anybuf, src=None)
            i = by_leader[src]
            bufs[i].copy_(anybuf)
            return i
        while True:
            for i in range(plan.g):
                if pending[i].is_completed():
                    pending[i].wait()                # orders the server stream after the receive
                    return i
            time.sleep(0)

    t = 0
    t0 = time.perf_counter()
    done = [False] * plan.g
    while t < max_updates:
        i = next_arrival()
        backend.sgd(W, V, bufs[i], snaps[i], hp_sum)
        t += 1
        events.append(AsyncEvent(i, read_step[i], t, t - 1 - read_step[i],
                                 time.perf_counter() - t0, drawn[i]))
        drawn[i] += 1
        snaps[i].copy_(W)                            # the group's next snapshot (and w_read)
        read_step[i] = t
        if t < max_updates:
            dist.send(go, dst=leaders[i], group=pair[i])
            dist.send(snaps[i], dst=leaders[i], group=pair[i])
            if nccl:
                pending[i] = dist.irecv(bufs[i], src=leaders[i], group=pair[i])
        else:
            dist.send(stop, dst=leaders[i], group=pair[i])   # its last gradient was applied
            done[i] = True
    if dev.type == "cuda":
        torch.cuda.synchronize(dev)
    seconds = time.perf_counter() - t0
    for _ in range(plan.g - sum(done)):              # drain: every other group gets a stop flag
        if nccl:
            i = next((j for j in range(plan.g) if not done[j]))
            pending[i].wait()
        else:
            i = by_leader[dist.recv(anybuf, src=None)]
        dist.send(stop, dst=leaders[i], group=pair[i])
        done[i] = True
    return AsyncResult(events, W, V, seconds)


def run_worker(plan: ExecutionPlan, backend, hp: Hyperparams, W0: torch.Tensor, n_examples: int,
               seed: int) -> int:
    """Ranks 1..N.  Returns how many gradients this rank's group produced."""
    rank = dist.get_rank()
    if rank == 0:
        raise RuntimeError("rank 0 is the server")
    intra, pair = _new_groups(plan)
    group = (rank - 1) // plan.k
    member = (rank - 1) % plan.k
    ranks = worker_ranks(plan, group)
    pg = intra[group]
    sg = pair[group]   # server <-> leader
    if hp.b % plan.k:
        raise ValueError(f"group batch b={hp.b} is not divisible by k={plan.k}")
    per = hp.b // plan.k
    rng = batch_stream(seed, group)
    W = W0.clone()
    flag = torch.zeros(1, dtype=torch.int32, device=W.device)
    n = 0
    while True:
        idx = rng.integers(0, n_examples, size=hp.b)
        G = backend.grad(W, idx[member * per:(member + 1) * per])
        if plan.k > 1:
            dist.all_reduce(G, group=pg)            # sum of k slice means
        if member == 0:
            dist.send(G, dst=0, group=sg)
            dist.recv(flag, src=0, group=sg)
        if plan.k > 1:
            dist.broadcast(flag, src=ranks[0], group=pg)
        n += 1
        if int(flag.item()) == 0:
            return n
        if member == 0:
            dist.recv(W, src=0, group=sg)
        if plan.k > 1:
            dist.broadcast(W, src=ranks[0], group=pg)


def replay(events: list, plan: ExecutionPlan, backend, hp: Hyperparams, W0: torch.Tensor,
           n_examples: int, seed: int) -> tuple[torch.Tensor, torch.Tensor]:
    """Re-apply an asynchronous run's update log in order on one device: the
    j-th update of group i uses the gradient of that group's j-th batch at the
    model the group had read (the state after write ``read_step``).  With k = 1
    and the same kernels this reproduces the run's final model bit for bit."""
    W = W0.clone()
    V = torch.zeros_like(W)
    hp_sum = hp.replace(eta=hp.eta / plan.k, lam=hp.lam * plan.k)
    rngs = [batch_stream(seed, i) for i in range(plan.g)]
    snaps = [W0.clone() for _ in range(plan.g)]
    per = hp.b // plan.k
    for e in events:
        idx = rngs[e.group_id].integers(0, n_examples, size=hp.b)
        G = None
        for m in range(plan.k):                      # the group's k slice gradients, summed
            Gm = backend.grad(snaps[e.group_id], idx[m * per:(m + 1) * per])
            G = Gm if G is None else G.add_(Gm)
        backend.sgd(W, V, G, snaps[e.group_id], hp_sum)
        snaps[e.group_id] = W.clone()
    return W, V
