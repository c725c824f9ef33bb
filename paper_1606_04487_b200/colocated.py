"""Free-running compute groups with the update server CO-LOCATED on rank 0
(the paper's mapping, cluster.py:54-73 / simulator.py:3-7:
N devices split into g groups of k = N/g, the serial model server living on
one of them -- no extra device).

Every rank is a worker: group i is ranks [i k, (i+1) k), its leader the first
of them.  Rank 0 is group 0's leader AND runs the update server in a second
host thread on its own CUDA stream:

* a group computes its gradient data parallel (k slice means, summed by an
  allreduce over the group's communicator), its leader DMAs the sum into its
  receive lane on rank 0 (copy engines over NVLink, IPC-mapped buffers),
  waits for the copy, then takes a ticket in the shared-memory mailbox
  (mailbox.cu);
* the server consumes tickets in order -- FIFO in order of arrival, like the
  reference's serial server -- applies V = mu V - eta (G + lam w_read);
  W += V with w_read = the snapshot that group computed on (stale_step,
  sgd.py:104-112), DMAs the new W into the group leader's model buffer and
  posts the snapshot sequence number;
* the leader (and every member, which watches the same mailbox slot) sees the
  sequence advance, the leader broadcasts the snapshot inside the group, and
  the next gradient starts.  No group ever waits for another group.

The 250 MB model and gradients never go through a collective library: they
move GPU to GPU by DMA; the only collectives are the group-internal
allreduce / broadcast, through the library's own C-ABI communicators
(comm.py, NCCL) -- torch.distributed only bootstraps (IPC handles, mailbox
name, NCCL unique id).  The update log is the same as async_groups' and
replays with ``async_groups.replay``.

``store="shm"`` swaps the IPC/DMA payload transport for host shared memory
and the C-ABI communicators for torch.distributed groups, so the same
protocol runs on CPU (gloo) in the multi-process tests.
"""

from __future__ import annotations

import ctypes
import os
import threading
import time
import uuid

import numpy as np
import torch
import torch.distributed as dist

from . import _abi
from .async_groups import AsyncEvent, AsyncResult
from .cluster import ExecutionPlan
from .sgd import Hyperparams, batch_stream

TIMEOUT_MS = 600_000


def group_of(plan: ExecutionPlan, rank: int) -> tuple[int, int]:
    """(group, member) of a global rank: groups of k consecutive ranks."""
    return rank // plan.k, rank % plan.k


# ----------------------------------------------------------- mailbox ----
class Mailbox:
    """The shared-memory ticket ring + snapshot sequence slots (mailbox.cu)."""

    def __init__(self, name: str, ngroups: int, create: bool):
        self.name = name
        self._box = ctypes.c_void_p()
        if create:
            _abi.call("omni_mailbox_create", name.encode(), ngroups, ctypes.byref(self._box))
        else:
            _abi.call("omni_mailbox_open", name.encode(), ctypes.byref(self._box), TIMEOUT_MS)
        self._owner = create

    def post(self, group: int) -> int:
        t = ctypes.c_longlong()
        _abi.call("omni_mailbox_post", self._box, group, ctypes.byref(t))
        return t.value

    def next(self) -> int:
        g = ctypes.c_int()
        _abi.call("omni_mailbox_next", self._box, ctypes.byref(g), TIMEOUT_MS)
        return g.value

    def snap_post(self, group: int, seq: int) -> None:
        _abi.call("omni_mailbox_snap_post", self._box, group, seq)

    def snap_wait(self, group: int, last: int) -> int:
        s = ctypes.c_longlong()
        _abi.call("omni_mailbox_snap_wait", self._box, group, last, ctypes.byref(s), TIMEOUT_MS)
        return s.value

    def close(self) -> None:
        if self._box:
            _abi.call("omni_mailbox_close", self._box, self.name.encode() if self._owner else None)
            self._box = ctypes.c_void_p()


# ------------------------------------------------------ payload stores --
class PeerStore:
    """GPU payloads: rank 0 holds one receive lane per group; every leader one
    model buffer the server writes snapshots into; both mapped across
    processes with CUDA IPC, moved with copy-engine DMA (omni_copy_async)."""

    def __init__(self, plan: ExecutionPlan, W0: torch.Tensor):
        from .comm import PeerUpdate

        rank = dist.get_rank()
        self.dev = W0.device
        self.n = W0.numel()
        self.esz = W0.element_size()
        self.plan = plan
        self.is_leader = rank % plan.k == 0
        self.lanes = torch.empty((plan.g, self.n), dtype=W0.dtype, device=self.dev) if rank == 0 else None
        self.model = W0.clone() if self.is_leader else None   # the leader's model (snapshot) buffer
        mine = {}
        if rank == 0:
            mine["lanes"] = PeerUpdate._handle(self.lanes)
        if self.is_leader:
            mine["model"] = PeerUpdate._handle(self.model)
        allh = [None] * dist.get_world_size()
        dist.all_gather_object(allh, mine)
        self._opened = {}
        self.lane_ptr = None
        if self.is_leader:
            gi = rank // plan.k
            if rank == 0:
                self.lane_ptr = self.lanes[gi].data_ptr()
            else:
                h, off = allh[0]["lanes"]
                self.lane_ptr = self._open(h, off) + gi * self.n * self.esz
        self.model_ptrs = None
        if rank == 0:
            self.model_ptrs = []
            for gi in range(plan.g):
                r = gi * plan.k
                if r == 0:
                    self.model_ptrs.append(self.model.data_ptr())
                else:
                    h, off = allh[r]["model"]
                    self.model_ptrs.append(self._open(h, off))

    def _open(self, h: bytes, off: int) -> int:
        if h not in self._opened:
            base = ctypes.c_void_p()
            _abi.call("omni_ipc_open", h, ctypes.byref(base))
            self._opened[h] = base.value
        return self._opened[h] + off

    def lane(self, gi: int) -> torch.Tensor:
        if gi == 0 and self.local_grad is not None:
            return self.local_grad
        return self.lanes[gi]

    local_grad = None   # rank 0's own group: the server reads its gradient buffer in place

    def push_grad(self, G: torch.Tensor) -> None:
        """Leader: G -> its lane on rank 0; returns once the copy has landed.
        On rank 0 itself the lane is G (zero copy: G stays untouched until
        this group's next snapshot has arrived)."""
        s = torch.cuda.current_stream(self.dev)
        if self.lanes is not None:   # rank 0, group 0
            self.local_grad = G
        else:
            _abi.call("omni_copy_async", ctypes.c_void_p(self.lane_ptr), ctypes.c_void_p(G.data_ptr()),
                      self.n * self.esz, ctypes.c_void_p(s.cuda_stream))
        s.synchronize()

    def push_snap(self, gi: int, W: torch.Tensor) -> None:
        """Server (rank 0, on its own stream): W -> group gi's leader model."""
        s = torch.cuda.current_stream(self.dev)
        _abi.call("omni_copy_async", ctypes.c_void_p(self.model_ptrs[gi]), ctypes.c_void_p(W.data_ptr()),
                  self.n * self.esz, ctypes.c_void_p(s.cuda_stream))
        s.synchronize()

    def close(self) -> None:
        for base in self._opened.values():
            _abi.call("omni_ipc_close", ctypes.c_void_p(base))
        self._opened.clear()


class ShmStore:
    """CPU payloads in host shared memory (the gloo tests)."""

    def __init__(self, plan: ExecutionPlan, W0: torch.Tensor):
        from multiprocessing import shared_memory

        rank = dist.get_rank()
        self.plan = plan
        self.n = W0.numel()
        dt = W0.numpy().dtype
        self.is_leader = rank % plan.k == 0
        self._shm = []
        names = {}
        if rank == 0:
            shm = shared_memory.SharedMemory(create=True, size=plan.g * self.n * dt.itemsize)
            self._shm.append(shm)
            self.lanes = torch.from_numpy(np.ndarray((plan.g, self.n), dtype=dt, buffer=shm.buf))
            names["lanes"] = shm.name
        self.model = None
        if self.is_leader:
            shm = shared_memory.SharedMemory(create=True, size=self.n * dt.itemsize)
            self._shm.append(shm)
            self.model = torch.from_numpy(np.ndarray((self.n,), dtype=dt, buffer=shm.buf))
            self.model.copy_(W0)
            names["model"] = shm.name
        alln = [None] * dist.get_world_size()
        dist.all_gather_object(alln, names)
        self._lane_view = None
        if self.is_leader:
            gi = rank // plan.k
            if rank == 0:
                self._lane_view = self.lanes[gi]
            else:
                shm = shared_memory.SharedMemory(name=alln[0]["lanes"])
                self._shm.append(shm)
                self._lane_view = torch.from_numpy(np.ndarray((plan.g, self.n), dtype=dt, buffer=shm.buf))[gi]
        self._models = None
        if rank == 0:
            self._models = []
            for gi in range(plan.g):
                r = gi * plan.k
                if r == 0:
                    self._models.append(self.model)
                else:
                    shm = shared_memory.SharedMemory(name=alln[r]["model"])
                    self._shm.append(shm)
                    self._models.append(torch.from_numpy(np.ndarray((self.n,), dtype=dt, buffer=shm.buf)))
        self._created = {v for v in names.values()}

    def lane(self, gi: int) -> torch.Tensor:
        return self.lanes[gi]

    def push_grad(self, G: torch.Tensor) -> None:
        self._lane_view.copy_(G)

    def push_snap(self, gi: int, W: torch.Tensor) -> None:
        self._models[gi].copy_(W)

    def close(self) -> None:
        for shm in self._shm:
            name = shm.name
            try:
                shm.close()
                if name in self._created:
                    shm.unlink()
            except Exception:   # noqa: BLE001
                pass
        self._shm = []


# ---------------------------------------------------- group collectives --
class _OmniGroup:
    """A compute group's allreduce / broadcast on the library's own NCCL
    communicators (comm.py, C-ABI): world communicator split by group."""

    def __init__(self, plan: ExecutionPlan, dev: torch.device):
        from . import comm

        rank, world = dist.get_rank(), dist.get_world_size()
        uid = [comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        self.world = comm.Communicator.init_rank(world, uid[0], rank, dev.index)
        gi, m = group_of(plan, rank)
        self.comm = self.world.split(gi, m)

    def allreduce_sum(self, t):
        self.comm.allreduce_sum(t)

    def broadcast(self, t, root_member: int):
        self.comm.broadcast(t, root_member)

    def close(self):
        self.comm.destroy()
        self.world.destroy()


class _TorchGroup:
    def __init__(self, plan: ExecutionPlan):
        rank = dist.get_rank()
        groups = [dist.new_group(list(range(i * plan.k, (i + 1) * plan.k))) for i in range(plan.g)]
        self.gi, _ = group_of(plan, rank)
        self.pg = groups[self.gi]
        self.root = self.gi * plan.k

    def allreduce_sum(self, t):
        dist.all_reduce(t, group=self.pg)

    def broadcast(self, t, root_member: int):
        dist.broadcast(t, src=self.root + root_member, group=self.pg)

    def close(self):
        pass


# ------------------------------------------------------------- runtime --
def run_colocated(plan: ExecutionPlan, backend, hp: Hyperparams, W0: torch.Tensor, n_examples: int,
                  seed: int, max_updates: int, store: str = "peer") -> AsyncResult | None:
    """Every rank calls this.  Rank 0 returns the update log and the final
    master model (AsyncResult); the others return None."""
    if plan.N != dist.get_world_size():
        raise ValueError(f"plan has N={plan.N} devices, the process group {dist.get_world_size()} ranks")
    if hp.b % plan.k:
        raise ValueError(f"group batch b={hp.b} is not divisible by k={plan.k}")
    rank = dist.get_rank()
    gi, member = group_of(plan, rank)
    name = [f"/omni_ag_{uuid.uuid4().hex[:16]}" if rank == 0 else None]
    dist.broadcast_object_list(name, src=0)
    box = Mailbox(name[0], plan.g, create=True) if rank == 0 else None
    dist.barrier()
    if rank != 0:
        box = Mailbox(name[0], plan.g, create=False)
    gpu = store == "peer"
    st = PeerStore(plan, W0) if gpu else ShmStore(plan, W0)
    grp = (_OmniGroup(plan, W0.device) if gpu else _TorchGroup(plan)) if plan.k > 1 else None
    dist.barrier()

    result = {}
    server = None
    if rank == 0:
        server = threading.Thread(target=_serve, args=(plan, backend, hp, W0, st, box, max_updates, result,
                                                       gpu), daemon=True)
        server.start()
    try:
        _work(plan, backend, hp, W0, st, box, grp, gi, member, n_examples, seed)
    finally:
        if server is not None:
            server.join()
        dist.barrier()
        if grp is not None:
            grp.close()
        st.close()
        box.close()
    if rank != 0:
        return None
    if "error" in result:
        raise result["error"]
    return result["res"]


def _work(plan, backend, hp, W0, st, box, grp, gi, member, n_examples, seed) -> int:
    """A worker: gradient at the group's current snapshot, group allreduce,
    leader pushes it to the server; wait for the next snapshot (or stop)."""
    per = hp.b // plan.k
    rng = batch_stream(seed, gi)
    W = st.model if member == 0 else W0.clone()
    last, n = 0, 0
    hooked = plan.k > 1 and isinstance(grp, _OmniGroup) and hasattr(backend, "grad_hooked")
    while True:
        idx = rng.integers(0, n_examples, size=hp.b)
        mine = idx[member * per:(member + 1) * per]
        if hooked:
            # each layer's slice of the group allreduce is issued on the weight-
            # gradient stream as soon as the layer is done, overlapping the rest
            # of the backward (the sum of the k slice means lands in engine.grad)
            G = backend.engine.grad
            backend.grad_hooked(W, mine, lambda lo, hi: grp.allreduce_sum(G[lo:hi]))
        else:
            G = backend.grad(W, mine)
            if plan.k > 1:
                grp.allreduce_sum(G)                   # sum of the k slice means
        if member == 0:
            st.push_grad(G)                            # landed in the server lane
            box.post(gi)
        last = box.snap_wait(gi, last)
        n += 1
        if last < 0:
            return n
        if plan.k > 1:
            grp.broadcast(W, 0)                        # leader's new snapshot to the group


def _serve(plan, backend, hp, W0, st, box, max_updates, result, gpu) -> None:
    """Rank 0's server thread: FIFO updates in ticket order (simulator.py:170-205)."""
    try:
        if gpu:
            torch.cuda.set_device(W0.device)           # the current device is per thread
        ctx = torch.cuda.stream(torch.cuda.Stream(device=W0.device)) if gpu else _Null()
        with ctx:
            W = W0.clone()
            V = torch.zeros_like(W)
            snaps = [W0.clone() for _ in range(plan.g)]   # what each group computes on (w_read)
            hp_sum = hp.replace(eta=hp.eta / plan.k, lam=hp.lam * plan.k)
            read_step = [0] * plan.g
            drawn = [0] * plan.g
            seq = [0] * plan.g
            events = []
            t = 0
            t0 = time.perf_counter()
            stopped = [False] * plan.g
            while t < max_updates:
                i = box.next()
                backend.sgd(W, V, st.lane(i), snaps[i], hp_sum)
                snaps[i].copy_(W)
                t += 1
                events.append(AsyncEvent(i, read_step[i], t, t - 1 - read_step[i],
                                         time.perf_counter() - t0, drawn[i]))
                drawn[i] += 1
                read_step[i] = t
                if t < max_updates:
                    st.push_snap(i, W)                  # waits for the DMA
                    seq[i] += 1
                    box.snap_post(i, seq[i])
                else:
                    if gpu:
                        torch.cuda.current_stream(W0.device).synchronize()
                    box.snap_post(i, -1)
                    stopped[i] = True
            seconds = time.perf_counter() - t0
            for _ in range(plan.g - sum(stopped)):      # every other group: its pending gradient, then stop
                i = box.next()
                box.snap_post(i, -1)
            result["res"] = AsyncResult(events, W, V, seconds)
    except Exception as e:   # noqa: BLE001  (re-raised on rank 0's main thread)
        result["error"] = e


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False
