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


# ----------------------------------------------------------- merged FC --
# The paper's physical mapping: the server also owns the
# fully connected layers.  A group runs its conv forward on its (stale)
# snapshot, ships the pool5 activations to the server, which runs the FC
# layers with the CURRENT FC model, updates it at once (FC staleness 0) and
# returns d(pool5); the group back-propagates the conv part and ships the conv
# gradient, which the server applies FIFO like above.  Groups of one GPU.

@dataclass(frozen=True)
class MergedEvent:
    kind: str            # "fc" (FC update from a group's activations) or "conv"
    group_id: int
    read_step: int       # conv model version the group computed on
    write_step: int      # conv model version after this event (conv events advance it)
    fc_step: int         # FC model version after this event
    arrive_time: float
    batch_index: int


def _split_buffers(eng, b):
    f = eng.first_fc
    return f, eng.ops[f].inp.value[:b], eng.ops[f].inp.grad[:b]


def run_server_merged(plan: ExecutionPlan, head, hp: Hyperparams, W0: torch.Tensor, fc_off: int,
                      act_shape: tuple, max_updates: int):
    """Rank 0 with merged FC.  ``head``: a GpuNet for the FC layers at the group
    batch with input_grad=True.  Returns (events, W, V, seconds)."""
    from . import kernels as K

    if plan.k != 1:
        raise ValueError("merged-FC asynchronous groups use one GPU per group (k = 1)")
    _, pair = _new_groups(plan)
    if dist.get_backend() != "nccl":
        raise RuntimeError("merged-FC asynchronous groups need NCCL (CUDA engines)")
    dev = W0.device
    W = W0.clone()
    V = torch.zeros_like(W)
    b = hp.b
    leaders = [worker_ranks(plan, i)[0] for i in range(plan.g)]
    acts = [torch.empty(act_shape, device=dev) for _ in range(plan.g)]
    labs = [torch.empty(b, dtype=torch.int32, device=dev) for _ in range(plan.g)]
    grads = [torch.empty(fc_off, device=dev) for _ in range(plan.g)]
    snaps = [W0[:fc_off].clone() for _ in range(plan.g)]
    read_step = [0] * plan.g
    drawn = [0] * plan.g
    phase = ["act"] * plan.g
    go = torch.ones(1, dtype=torch.int32, device=dev)
    stop = torch.zeros(1, dtype=torch.int32, device=dev)

    def post(i):
        if phase[i] == "act":
            return [dist.irecv(acts[i], src=leaders[i], group=pair[i]),
                    dist.irecv(labs[i], src=leaders[i], group=pair[i])]
        return [dist.irecv(grads[i], src=leaders[i], group=pair[i])]

    pending = [post(i) for i in range(plan.g)]
    events = []
    t = fc_t = 0
    t0 = time.perf_counter()
    # the head stages its weights from a 16-byte aligned vector (TMA): when the
    # FC parameters do not start on a 4-float boundary (LeNet: fc_off % 4 = 2)
    # the server keeps them in their own aligned buffers and writes them back
    # into W / V when it returns
    aligned = fc_off % 4 == 0
    Wfc = W[fc_off:] if aligned else W[fc_off:].clone()
    Vfc = V[fc_off:] if aligned else V[fc_off:].clone()
    while t < max_updates:
        i = None
        while i is None:
            for j in range(plan.g):
                if all(w.is_completed() for w in pending[j]):
                    i = j
                    break
            if i is None:
                time.sleep(0)
        for w in pending[i]:
            w.wait()
        if phase[i] == "act":                       # FC phase for group i, current FC model
            head.input.value[:b].copy_(acts[i])
            head.labels[:b].copy_(labs[i])
            head.forward(Wfc, b)
            head.backward(b)
            K.sgd_momentum(Wfc, Vfc, head.grad, Wfc, hp.eta, hp.mu, hp.lam)
            fc_t += 1
            events.append(MergedEvent("fc", i, read_step[i], t, fc_t, time.perf_counter() - t0,
                                      drawn[i]))
            dist.send(head.input.grad[:b].contiguous(), dst=leaders[i], group=pair[i])
            phase[i] = "grad"
        else:                                        # conv update, FIFO, stale snapshot
            K.sgd_momentum(W[:fc_off], V[:fc_off], grads[i], snaps[i], hp.eta, hp.mu, hp.lam)
            t += 1
            events.append(MergedEvent("conv", i, read_step[i], t, fc_t, time.perf_counter() - t0,
                                      drawn[i]))
            drawn[i] += 1
            snaps[i].copy_(W[:fc_off])
            read_step[i] = t
            phase[i] = "act"
            if t < max_updates:
                dist.send(go, dst=leaders[i], group=pair[i])
                dist.send(snaps[i], dst=leaders[i], group=pair[i])
            else:
                dist.send(stop, dst=leaders[i], group=pair[i])
                pending[i] = []
                continue
        pending[i] = post(i)
    torch.cuda.synchronize(dev)
    seconds = time.perf_counter() - t0
    # drain: finish every other group's current iteration, then stop it
    for i in range(plan.g):
        if not pending[i]:
            continue
        while True:
            for w in pending[i]:
                w.wait()
            if phase[i] == "act":                   # serve its FC phase without updating
                head.input.value[:b].copy_(acts[i])
                head.labels[:b].copy_(labs[i])
                head.forward(Wfc, b)
                head.backward(b)
                dist.send(head.input.grad[:b].contiguous(), dst=leaders[i], group=pair[i])
                phase[i] = "grad"
                pending[i] = post(i)
                continue
            dist.send(stop, dst=leaders[i], group=pair[i])
            break
    if not aligned:
        W[fc_off:].copy_(Wfc)
        V[fc_off:].copy_(Vfc)
    return events, W, V, seconds


def run_worker_merged(plan: ExecutionPlan, eng, problem, hp: Hyperparams, W0: torch.Tensor,
                      fc_off: int, seed: int) -> int:
    """Ranks 1..g (one GPU per group): conv forward -> activations to the
    server -> d(pool5) back -> conv backward -> conv gradient to the server."""
    rank = dist.get_rank()
    _, pair = _new_groups(plan)
    group = rank - 1
    sg = pair[group]
    b = hp.b
    rng = batch_stream(seed, group)
    W = W0.clone()
    f, act, dact = _split_buffers(eng, b)
    flag = torch.zeros(1, dtype=torch.int32, device=W.device)
    n = 0
    while True:
        idx = torch.from_numpy(rng.integers(0, problem._n, size=b)).to(W.device)
        eng.gather_batch(problem.data, problem.data_labels, idx)
        eng.forward(W, b, stop=f)
        dist.send(act.contiguous(), dst=0, group=sg)
        dist.send(eng.labels[:b].contiguous(), dst=0, group=sg)
        dist.recv(dact, src=0, group=sg)
        eng.backward(b, start=f)
        dist.send(eng.grad[:fc_off].contiguous(), dst=0, group=sg)
        dist.recv(flag, src=0, group=sg)
        n += 1
        if int(flag.item()) == 0:
            return n
        dist.recv(W[:fc_off], src=0, group=sg)


def replay_merged(events: list, plan: ExecutionPlan, eng, head, problem, hp: Hyperparams,
                  W0: torch.Tensor, fc_off: int, seed: int):
    """Re-apply a merged-FC run's log in order on one device (bit-exact: same
    kernels, same batches; a group's conv forward is recomputed from its
    snapshot before its backward)."""
    from . import kernels as K

    b = hp.b
    W = W0.clone()
    V = torch.zeros_like(W)
    aligned = fc_off % 4 == 0                        # (see run_server_merged)
    Wfc = W[fc_off:] if aligned else W[fc_off:].clone()
    Vfc = V[fc_off:] if aligned else V[fc_off:].clone()
    rngs = [batch_stream(seed, i) for i in range(plan.g)]
    snaps = [W0.clone() for _ in range(plan.g)]      # full-size vectors; conv part used
    idx_of = {}
    dacts = {}
    f, act, dact = _split_buffers(eng, b)
    for e in events:
        i = e.group_id
        if e.kind == "fc":
            idx = torch.from_numpy(rngs[i].integers(0, problem._n, size=b)).to(W.device)
            idx_of[i] = idx
            eng.gather_batch(problem.data, problem.data_labels, idx)
            eng.forward(snaps[i], b, stop=f)
            head.input.value[:b].copy_(act)
            head.labels[:b].copy_(eng.labels[:b])
            head.forward(Wfc, b)
            head.backward(b)
            K.sgd_momentum(Wfc, Vfc, head.grad, Wfc, hp.eta, hp.mu, hp.lam)
            dacts[i] = head.input.grad[:b].clone()
        else:
            eng.gather_batch(problem.data, problem.data_labels, idx_of[i])
            eng.forward(snaps[i], b, stop=f)
            dact.copy_(dacts[i])
            eng.backward(b, start=f)
            K.sgd_momentum(W[:fc_off], V[:fc_off], eng.grad[:fc_off], snaps[i][:fc_off],
                           hp.eta, hp.mu, hp.lam)
            snaps[i][:fc_off].copy_(W[:fc_off])
    if not aligned:
        W[fc_off:].copy_(Wfc)
        V[fc_off:].copy_(Vfc)
    return W, V
