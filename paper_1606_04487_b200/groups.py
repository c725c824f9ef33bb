"""Compute groups across GPUs: g groups of k = N/g ranks (one process per GPU).

Semantics are the reference's deterministic schedule (simulator.py:123-213
with service_mode="deterministic", cluster.py:54-73), which is strict round
robin: write step t >= 1 is made by group (t-1) mod g with the gradient of
draw floor((t-1)/g) of that group's batch stream, evaluated at the model
W(max(0, t-g)) -- the state right after the group's own previous write
(SURVEY.md section 3(C)).  That makes g updates per round independent, so
they run concurrently:

  round r, on every rank of group i:
    1. gradient at the group's snapshot on this rank's slice of the group batch
       (data parallel inside the group: k ranks x b/k images);
    2. allreduce (sum) inside the group -> the group gradient (mean over b);
    3. all-gather across groups (one rank per group per member index) ->
       G_0 .. G_{g-1} on every rank;
    4. replay the g momentum updates in group order (sgd.py:104-112: the
       regulariser also uses the writer's snapshot), keeping W after update i
       as group i's next snapshot.

Every rank therefore holds the master model and all g snapshots; no rank
waits on another except in the two collectives.  g = 1 degenerates to
synchronous data-parallel SGD with one allreduce per step.

The gradient/update provider is pluggable: ``CudaBackend`` (the B200 engine,
NCCL) is the product path; tests plug a CPU backend into the same runtime to
check the collective logic with gloo.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Protocol

import numpy as np
import torch
import torch.distributed as dist

from .cluster import ExecutionPlan
from .sgd import Hyperparams, batch_stream


class Backend(Protocol):
    device: torch.device

    def grad(self, W: torch.Tensor, idx: np.ndarray) -> torch.Tensor:
        """Mean-over-batch gradient at W of the examples ``idx`` (a fresh tensor)."""

    def sgd(self, W: torch.Tensor, V: torch.Tensor, G: torch.Tensor, w_read: torch.Tensor,
            hp: Hyperparams) -> None:
        """In place: V = mu V - eta (G + lam w_read); W += V."""

    def group_updates(self, rows: torch.Tensor, members: list, W: torch.Tensor, V: torch.Tensor,
                      snaps: list, hp: Hyperparams) -> None:
        """The g ordered updates of a round on one shard: for i in order, G_i =
        sum of rows[members[i]] (in that order), sgd(W, V, G_i, snaps[i]),
        then snaps[i] = W."""

    def exchange(self, plan: ExecutionPlan):
        """The runtime's collectives (comm.GroupExchange's methods)."""


class CudaBackend:
    """B200 engine: device gather + fused forward/backward + K8 update."""

    def __init__(self, problem, batch: int):
        self.problem = problem
        self.device = problem.device
        self.engine = problem.engine(batch)

    def grad(self, W, idx):
        from .problems import Batch

        b = self.problem.load_batch(self.engine, Batch(self.problem, idx))
        _, G = self.engine.loss_and_grad(W, b)
        return G.clone()

    def sgd(self, W, V, G, w_read, hp):
        from . import kernels as K

        K.sgd_momentum(W, V, G, w_read, hp.eta, hp.mu, hp.lam)

    def group_updates(self, rows, members, W, V, snaps, hp):
        from . import kernels as K

        K.group_updates(rows, members, W, V, snaps, hp.eta, hp.mu, hp.lam)

    def exchange(self, plan):
        from .comm import GroupExchange

        return GroupExchange(plan, self.device)

    def layer_ranges(self) -> list:
        """Parameter ranges [lo, hi) of the layers, in backward order (the
        order the engine's on_grad hook reports them)."""
        out = []
        for op in reversed(self.engine.ops):
            if op.kind in ("conv", "fc"):
                hi = op.boff + op.layer.d_out if op.boff >= 0 else op.woff + op.wsz
                out.append((op.woff, hi))
        return out

    def grad_fused(self, W, idx, fused_update) -> None:
        """Gradient into self.engine.grad with fused_update(lo, hi, stream)
        called on the engine's update stream as each layer's gradient is final
        and its data gradient no longer reads W (peer-memory rounds)."""
        from .problems import Batch

        b = self.problem.load_batch(self.engine, Batch(self.problem, idx))
        self.engine.forward(W, b)
        self.engine.backward(b, update=(W, W, W, 0.0, 0.0, 0.0), fused_update=fused_update)

    def grad_hooked(self, W, idx, on_grad) -> None:
        """Gradient with on_grad(lo, hi) called as each layer's gradient is
        enqueued (for overlapped per-layer exchanges); the gradient stays in
        self.engine.grad."""
        from .problems import Batch

        b = self.problem.load_batch(self.engine, Batch(self.problem, idx))
        self.engine.forward(W, b)
        self.engine.backward(b, on_grad=on_grad)


@dataclass(frozen=True)
class GroupEvent:
    group_id: int
    read_step: int
    write_step: int
    staleness: int


class GroupRuntime:
    def __init__(self, plan: ExecutionPlan, backend: Backend, hp: Hyperparams, W0: torch.Tensor,
                 n_examples: int, seed: int, sharded: bool = True, overlap: bool = False,
                 p2p: bool = False):
        if not dist.is_initialized():
            raise RuntimeError("GroupRuntime needs torch.distributed initialised (one rank per GPU)")
        world, rank = dist.get_world_size(), dist.get_rank()
        if plan.N != world:
            raise ValueError(f"plan.N={plan.N} != world size {world}")
        if hp.b % plan.k:
            raise ValueError(f"group batch b={hp.b} is not divisible by k={plan.k}")
        self.plan, self.backend, self.hp = plan, backend, hp
        self.rank = rank
        self.group = plan.group_of(rank)
        self.member = plan.member_of(rank)
        self.n_examples = n_examples
        self._x = None                       # collectives (backend.exchange), made on first use
        self.sharded = bool(sharded)
        self._layered = False
        self.snap_step = [0] * plan.g
        self.t = 0
        self.rng = batch_stream(seed, self.group)
        self.events: list[GroupEvent] = []
        self.dim = W0.numel()
        self._p2p = bool(p2p) and hasattr(backend, "grad_fused")
        if self._p2p:
            self._init_p2p(W0)
        elif self.sharded:
            # rank r owns elements [r*S, (r+1)*S) of W, V and of every group's snapshot
            N = world
            S = -(-self.dim // N)
            S = -(-S // 4) * 4                     # 16-byte aligned shards
            self._S = S
            lo, hi = rank * S, min((rank + 1) * S, self.dim)
            self._W = torch.zeros(S, dtype=W0.dtype, device=W0.device)
            self._W[:max(0, hi - lo)] = W0[lo:hi]
            self._V = torch.zeros_like(self._W)
            self._snapsh = [self._W.clone() for _ in range(plan.g)]
            self._snap_own = W0.clone()              # this rank's group snapshot, full length
            self._Gpad = torch.zeros(N * S, dtype=W0.dtype, device=W0.device)
            self._rows = torch.empty(N, S, dtype=W0.dtype, device=W0.device)
            self._back = torch.empty(N * S, dtype=W0.dtype, device=W0.device)
            self._layered = bool(overlap) and hasattr(backend, "grad_hooked")
            if self._layered:
                self._init_layered(W0)
        else:
            self._W = W0.clone()
            self._V = torch.zeros_like(self._W)
            self.snaps = [self._W.clone() for _ in range(plan.g)]
            self._gather = torch.empty(plan.g, self.dim, dtype=W0.dtype, device=W0.device)
        # gradients arrive as the SUM of k slice means; fold the 1/k into the fused
        # update: eta (G/k + lam w) = (eta/k) (G + k lam w)
        self._hp_sum = hp.replace(eta=hp.eta / plan.k, lam=hp.lam * plan.k)

    @property
    def x(self):
        """The collectives (the backend's exchange: the library's NCCL
        communicators on the CUDA backend).  Made on first use -- every rank
        reaches it in the same round -- so a peer-memory runtime that never
        assembles the master model opens no communicator."""
        if self._x is None:
            self._x = self.backend.exchange(self.plan)
        return self._x

    def _members(self) -> list:
        return [list(self.plan.group_ranks(i)) for i in range(self.plan.g)]

    def _log_round(self) -> None:
        for i in range(self.plan.g):
            self.t += 1
            self.events.append(GroupEvent(i, self.snap_step[i], self.t, self.t - 1 - self.snap_step[i]))
            self.snap_step[i] = self.t

    def _init_p2p(self, W0: torch.Tensor) -> None:
        """Peer-memory rounds (comm.PeerUpdate, copy-engine DMA): rank r owns
        part r of every layer slice (comm.owned_part) of W, V and of the g
        snapshots, kept in full-length buffers; each member's own-group
        snapshot buffer is mapped into every owner, which writes its parts."""
        from .comm import PeerUpdate

        self.sharded = True
        self._layers = self.backend.layer_ranges()
        self._Wf = W0.clone()
        self._Vf = torch.zeros_like(W0)
        self._snapf = [W0.clone() for _ in range(self.plan.g)]
        self._snap_own = W0.clone()
        self._peer = PeerUpdate(self.backend.engine.grad, self._snap_own, len(self._layers),
                                dist.group.WORLD, mode="dma")

    def _round_p2p(self) -> None:
        """One round with every exchange over NVLink peer memory, per layer as
        the backward produces it: gradient parts DMA'd to their owners, the g
        ordered updates of each owner's part (sum of the group's k lanes in
        member order, w_read = that group's snapshot), and the new snapshot
        parts DMA'd into the group members' snapshot buffers."""
        import ctypes

        from . import _abi
        from .comm import owned_part

        plan, N, peer = self.plan, self.plan.N, self._peer
        idx = self.rng.integers(0, self.n_examples, size=self.hp.b)
        hp = self._hp_sum
        esz = self._Wf.element_size()
        lanes = [[peer.g_lanes[m] for m in plan.group_ranks(i)] for i in range(plan.g)]
        lanes = [(ctypes.c_void_p * len(l))(*l) for l in lanes]
        wloc = (ctypes.c_void_p * plan.k)(self._Wf.data_ptr(), *([None] * (plan.k - 1)))
        V, Wf = self._Vf, self._Wf

        def fused(lo, hi, stream):
            s = ctypes.c_void_p(stream.cuda_stream)
            slot = peer.slot
            peer.slot += 1
            for p in range(N):                                  # my gradient parts -> owners
                if p != self.rank:
                    a, b = owned_part(lo, hi, N, p)
                    _abi.call("omni_copy_async",
                              ctypes.c_void_p(peer.r_ptrs[p] + self.rank * peer._lane + a * esz),
                              ctypes.c_void_p(peer.G.data_ptr() + a * esz), (b - a) * esz, s)
            _abi.call("omni_p2p_signal", peer.f_ptrs, N, self.rank, peer.GRAD_READY, slot,
                      peer.max_slots, peer._sp, s)
            _abi.call("omni_p2p_wait", ctypes.c_void_p(peer.flags.data_ptr()), N, self.rank,
                      peer.GRAD_READY, slot, slot + 1, peer.max_slots, peer._sp, s)
            a, b = owned_part(lo, hi, N, self.rank)
            if b > a:
                for i in range(plan.g):                         # the g ordered updates
                    snap = self._snapf[i]
                    _abi.call("omni_p2p_reduce_sgd_f32", lanes[i], wloc, plan.k, 0, a, b,
                              ctypes.c_void_p(V.data_ptr()), ctypes.c_void_p(snap.data_ptr()),
                              float(hp.eta), float(hp.mu), float(hp.lam), s)
                    _abi.call("omni_copy_async", ctypes.c_void_p(snap.data_ptr() + a * esz),
                              ctypes.c_void_p(Wf.data_ptr() + a * esz), (b - a) * esz, s)
                    for m in plan.group_ranks(i):               # group i reads W(t) next round
                        _abi.call("omni_copy_async", ctypes.c_void_p(peer.w_ptrs[m] + a * esz),
                                  ctypes.c_void_p(Wf.data_ptr() + a * esz), (b - a) * esz, s)
            _abi.call("omni_p2p_signal", peer.f_ptrs, N, self.rank, peer.W_DONE, slot,
                      peer.max_slots, peer._sp, s)

        peer.begin_step()
        self.backend.grad_fused(self._snap_own, self._my_slice(idx), fused)
        peer.finish()
        for i in range(plan.g):
            self.t += 1
            self.events.append(GroupEvent(i, self.snap_step[i], self.t, self.t - 1 - self.snap_step[i]))
            self.snap_step[i] = self.t

    def _assemble(self, full: torch.Tensor) -> torch.Tensor:
        """Peer-memory mode: the owners' parts of a full-length buffer, summed
        over ranks (every other element zeroed first: exact)."""
        from .comm import owned_part

        out = torch.zeros_like(full)
        for lo, hi in self._layers:
            a, b = owned_part(lo, hi, self.plan.N, self.rank)
            out[a:b] = full[a:b]
        self.x.world_allreduce(out)
        return out

    def _init_layered(self, W0: torch.Tensor) -> None:
        """Layer-aligned shards: every layer's range [lo, hi) is split into N
        pieces of q = ceil(len/N); rank r owns piece r of every layer, so each
        layer's gradient can be exchanged (all-to-all) as soon as it exists."""
        N, r = self.plan.N, self.rank
        dev = W0.device
        self._layers = []                 # (lo, hi, q, shard offset), backward order
        off = 0
        for lo, hi in self.backend.layer_ranges():
            q = -(-(hi - lo) // N)
            self._layers.append((lo, hi, q, off))
            off += q
        S = off
        self._S = S
        # gather index: full vector element -> position in the (N, S) array of shards
        gidx = torch.empty(self.dim, dtype=torch.int64)
        for lo, hi, q, o in self._layers:
            e = torch.arange(hi - lo)
            gidx[lo:hi] = (e // q) * S + o + (e % q)
        self._gidx = gidx.to(dev)
        sh = torch.zeros(S, dtype=W0.dtype, device=dev)
        for lo, hi, q, o in self._layers:
            a, z = lo + r * q, min(lo + (r + 1) * q, hi)
            if z > a:
                sh[o:o + (z - a)] = W0[a:z]
        self._W = sh
        self._V = torch.zeros_like(sh)
        self._snapsh = [sh.clone() for _ in range(self.plan.g)]
        self._send = {lo: torch.zeros(N * q, dtype=W0.dtype, device=dev) for lo, hi, q, o in self._layers}
        self._recv = {lo: torch.empty(N * q, dtype=W0.dtype, device=dev) for lo, hi, q, o in self._layers}
        self._back = torch.empty(N * S, dtype=W0.dtype, device=dev)

    def _full(self, shard: torch.Tensor) -> torch.Tensor:
        out = torch.empty(self.plan.N * shard.numel(), dtype=shard.dtype, device=shard.device)
        self.x.world_allgather(shard, out)
        if getattr(self, "_layered", False):
            return out[self._gidx]
        return out[:self.dim]

    @property
    def W(self) -> torch.Tensor:
        """The master model (sharded runtime: assembled from every rank's shard,
        a collective -- every rank calls it)."""
        if self._p2p:
            return self._assemble(self._Wf)
        return self._full(self._W) if self.sharded else self._W

    @property
    def V(self) -> torch.Tensor:
        if self._p2p:
            return self._assemble(self._Vf)
        return self._full(self._V) if self.sharded else self._V

    def _my_slice(self, idx: np.ndarray) -> np.ndarray:
        per = self.hp.b // self.plan.k
        return idx[self.member * per:(self.member + 1) * per]

    def run(self, rounds: int) -> None:
        for _ in range(rounds):
            self.round()

    def close(self) -> None:
        """Release the communicators and peer mappings (collective: every rank)."""
        if self._x is not None and hasattr(self._x, "close"):
            self._x.close()
            self._x = None
        if self._p2p and getattr(self, "_peer", None) is not None:
            self._peer.close()
            self._peer = None

    def round(self) -> None:
        """One round = g master updates, one per group, in group order."""
        if self._p2p:
            return self._round_p2p()
        if self.sharded:
            return self._round_layered() if self._layered else self._round_sharded()
        plan = self.plan
        idx = self.rng.integers(0, self.n_examples, size=self.hp.b)
        G = self.backend.grad(self.snaps[self.group], self._my_slice(idx))
        if plan.k > 1:
            self.x.group_allreduce(G)                       # sum of k slice means
        if plan.g > 1:
            self.x.cross_allgather(G, self._gather)         # row i = group i's gradient
            rows = self._gather
        else:
            rows = G.view(1, -1)
        # the g ordered updates; snaps[i] <- W after update i (group i reads it next round)
        self.backend.group_updates(rows, [[i] for i in range(plan.g)], self._W, self._V, self.snaps,
                                   self._hp_sum)
        self._log_round()

    def _round_layered(self) -> None:
        """_round_sharded with layer-aligned shards: each layer's gradient
        all-to-all is issued from the backward's on_grad hook on the exchange's
        own stream, overlapping the rest of the backward; the g ordered
        updates of each layer's shard (one kernel per layer) and the snapshot
        exchange are as in _round_sharded."""
        plan, N = self.plan, self.plan.N
        idx = self.rng.integers(0, self.n_examples, size=self.hp.b)
        works = []
        G = self.backend.engine.grad
        lens = {lo: hi - lo for lo, hi, q, o in self._layers}

        def hook(lo, hi):
            send = self._send[lo]
            send[:lens[lo]].copy_(G[lo:hi])                    # (on the gradient's stream)
            works.append(self.x.all_to_all_async(list(send.view(N, -1)), self._recv[lo]))

        self.backend.grad_hooked(self._snap_own, self._my_slice(idx), hook)
        for w in works:
            w.wait()
        members = self._members()
        for lo, hi, q, o in self._layers:
            self.backend.group_updates(self._recv[lo].view(N, q), members, self._W[o:o + q],
                                       self._V[o:o + q], [s[o:o + q] for s in self._snapsh],
                                       self._hp_sum)
        self._log_round()
        self.x.all_to_all([self._snapsh[plan.group_of(m)] for m in range(N)], self._back)
        self._snap_own = self._back[self._gidx]

    def _round_sharded(self) -> None:
        """The same round with the update work partitioned: one all-to-all gives
        every rank its shard of each group's gradient, one kernel applies the g
        ordered updates to this rank's shard of W, V and of the g snapshots
        (group i's gradient = the sum of its members' rows in member order),
        and a second all-to-all returns to every rank its own group's next
        snapshot.  Per-rank traffic ~2 models per round (vs a group allreduce
        plus g models gathered), update work g/N models (vs g)."""
        plan, N, S = self.plan, self.plan.N, self._S
        idx = self.rng.integers(0, self.n_examples, size=self.hp.b)
        G = self.backend.grad(self._snap_own, self._my_slice(idx))
        self._Gpad[:self.dim].copy_(G)
        rows = self._rows
        self.x.all_to_all(list(self._Gpad.view(N, S)), rows.view(-1))   # row m = rank m's gradient, my shard
        self.backend.group_updates(rows, self._members(), self._W, self._V, self._snapsh, self._hp_sum)
        self._log_round()
        self.x.all_to_all([self._snapsh[plan.group_of(m)] for m in range(N)], self._back)
        self._snap_own = self._back[:self.dim]            # my group's next snapshot (a view)
