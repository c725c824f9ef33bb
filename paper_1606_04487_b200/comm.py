"""NCCL communicators through the C-ABI (include/omni.h, "comm" section).

The reference's multi-GPU semantics are logical (one process; the g groups of
``ExecutionPlan`` are simulated, cluster.py:54-73, simulator.py:3-7).  The
runtimes in this package (``problems.DeviceSession`` at N > 1, ``groups``,
``async_groups``) use ``torch.distributed`` for the plumbing; this module is
the same transport for a host that binds only libomni.so: one communicator
per process (``init_rank``) or per device of one process (``init_all``),
``split`` into compute groups, an in-place gradient ``allreduce_sum`` and the
point-to-point snapshot / gradient transfers of the update server.

Buffers are CUDA float32 tensors (only their pointers cross the ABI); every
call is asynchronous on the given stream (default: torch's current stream).
"""

from __future__ import annotations

import ctypes

import torch

from . import _abi

ID_BYTES = 128
SPLIT_NOCOLOR = -1


def nccl_version() -> int:
    v = ctypes.c_int()
    _abi.call("omni_comm_nccl_version", ctypes.byref(v))
    return v.value


def unique_id() -> bytes:
    """A fresh NCCL unique id (rank 0 makes it; the host ships it to the others)."""
    buf = ctypes.create_string_buffer(ID_BYTES)
    _abi.call("omni_comm_unique_id", buf)
    return buf.raw


def _stream(stream, t: torch.Tensor):
    s = stream if stream is not None else torch.cuda.current_stream(t.device)
    return ctypes.c_void_p(s.cuda_stream)


def _buf(t: torch.Tensor) -> ctypes.c_void_p:
    if not t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous():
        raise ValueError("communicator buffers must be contiguous CUDA float32 tensors")
    return ctypes.c_void_p(t.data_ptr())


class Communicator:
    """One NCCL communicator (an opaque ``ncclComm_t`` owned by this object)."""

    def __init__(self, handle: int, device: int):
        self._h = ctypes.c_void_p(handle)
        self.device = device

    @classmethod
    def init_rank(cls, nranks: int, uid: bytes, rank: int, device: int) -> "Communicator":
        if len(uid) != ID_BYTES:
            raise ValueError(f"unique id must be {ID_BYTES} bytes")
        h = ctypes.c_void_p()
        _abi.call("omni_comm_init_rank", ctypes.byref(h), nranks, uid, rank, device)
        return cls(h.value, device)

    @classmethod
    def init_all(cls, devices: list[int]) -> list["Communicator"]:
        n = len(devices)
        devs = (ctypes.c_int * n)(*devices)
        hs = (ctypes.c_void_p * n)()
        _abi.call("omni_comm_init_all", n, devs, hs)
        return [cls(hs[i], devices[i]) for i in range(n)]

    @property
    def handle(self) -> int:
        return self._h.value or 0

    def size_rank(self) -> tuple[int, int]:
        s, r = ctypes.c_int(), ctypes.c_int()
        _abi.call("omni_comm_size_rank", self._h, ctypes.byref(s), ctypes.byref(r))
        return s.value, r.value

    @property
    def size(self) -> int:
        return self.size_rank()[0]

    @property
    def rank(self) -> int:
        return self.size_rank()[1]

    def split(self, color: int, key: int) -> "Communicator":
        """Ranks with the same color form one communicator ordered by key
        (one compute group of the plan); SPLIT_NOCOLOR opts out (the result's
        handle stays 0).  Collective; inside ``group()`` NCCL fills the handle
        at group exit, so the returned object owns the slot it writes."""
        sub = Communicator(0, self.device)
        _abi.call("omni_comm_split", self._h, color, key, ctypes.byref(sub._h))
        return sub

    def allreduce_sum(self, t: torch.Tensor, stream=None) -> torch.Tensor:
        _abi.call("omni_allreduce_sum_f32", self._h, _buf(t), t.numel(), _stream(stream, t))
        return t

    def broadcast(self, t: torch.Tensor, root: int, stream=None) -> torch.Tensor:
        _abi.call("omni_broadcast_f32", self._h, _buf(t), t.numel(), root, _stream(stream, t))
        return t

    def send(self, t: torch.Tensor, peer: int, stream=None) -> None:
        _abi.call("omni_send_f32", self._h, _buf(t), t.numel(), peer, _stream(stream, t))

    def recv(self, t: torch.Tensor, peer: int, stream=None) -> torch.Tensor:
        _abi.call("omni_recv_f32", self._h, _buf(t), t.numel(), peer, _stream(stream, t))
        return t

    def allgather(self, t: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
        """out[r*n:(r+1)*n] = rank r's t (n = t.numel())."""
        if out.numel() < t.numel() * self.size or not out.is_contiguous():
            raise ValueError("allgather: out must be contiguous with nranks * t.numel() elements")
        _abi.call("omni_allgather_f32", self._h, _buf(t), _buf(out), t.numel(), _stream(stream, t))
        return out

    def all_to_all(self, parts: list, recv: torch.Tensor, stream=None) -> torch.Tensor:
        """parts[m] (n floats each, anywhere in device memory) -> rank m;
        rank m's part for this rank -> recv[m*n:(m+1)*n]."""
        n = parts[0].numel()
        if len(parts) != self.size or any(p.numel() != n or not p.is_contiguous() for p in parts):
            raise ValueError("all_to_all: one contiguous part of equal length per rank")
        if recv.numel() < n * len(parts) or not recv.is_contiguous():
            raise ValueError("all_to_all: recv must be contiguous with nranks * n elements")
        ptrs = (ctypes.c_void_p * len(parts))(*[p.data_ptr() for p in parts])
        _abi.call("omni_all_to_all_f32", self._h, ptrs, _buf(recv), n, _stream(stream, recv))
        return recv

    def destroy(self) -> None:
        if self._h.value:
            _abi.call("omni_comm_destroy", self._h)
            self._h = ctypes.c_void_p()


class group:
    """``with comm.group(): ...`` fuses the enclosed send/recv calls (ncclGroupStart/End)."""

    def __enter__(self):
        _abi.call("omni_comm_group_start")
        return self

    def __exit__(self, *exc):
        _abi.call("omni_comm_group_end")
        return False


def owned_part(lo: int, hi: int, n: int, rank: int) -> tuple[int, int]:
    """Rank ``rank``'s elements of the slice [lo, hi) in the peer-memory update:
    contiguous chunks of c = 4*ceil((hi-lo)/(4n)) (whole float4s), the last
    ones clipped (possibly empty)."""
    c = 4 * -(-(hi - lo) // (4 * n))
    a = min(hi, lo + rank * c)
    return a, min(hi, a + c)


class PeerUpdate:
    """Fused gradient allreduce + momentum update over peer memory
    (include/omni.h "p2p"): data parallelism without a collective library on
    the data path.  One instance per rank of a torch.distributed group (used
    only to swap IPC handles once).

    Each rank owns 1/N of every layer slice (``owned_part``).  Per step:
    ``begin_step()`` advances the device step counter; per layer slice, once
    the slice's gradient is final and its data gradient no longer reads W,
    ``layer(lo, hi, ...)`` (on the update stream) moves the gradient parts to
    their owners, signals, waits for every rank's signal, runs the fused
    reduce + momentum update on this rank's part, and sends the new W part
    to every rank; ``finish()`` holds the stream until every rank's W parts
    have landed.  Two transports:

    * ``"dma"`` (default): the NVLink transfers are copy-engine DMAs
      (``omni_copy_async`` into the owners' receive lanes ``R`` and into the
      peers' W) -- no SM is taken from the persistent GEMM grids running
      beside them; the kernel reads only local HBM;
    * ``"pull"``: the kernel itself loads the peers' gradients and stores W
      into the peers over NVLink (faster alone, 0.65 vs 1.1 ms per 250 MB at
      N = 4, but it competes with the backward's GEMMs for SMs).

    V is valid only on each element's owner until ``gather_momentum()``.
    Step numbers live on the device, so a CUDA graph of the whole step
    replays correctly."""

    GRAD_READY, W_DONE = 0, 1

    def __init__(self, G: torch.Tensor, W: torch.Tensor, max_slots: int, process_group=None,
                 mode: str = "dma"):
        import torch.distributed as dist

        if mode not in ("pull", "dma"):
            raise ValueError("mode must be 'pull' (SM loads/stores over NVLink) or 'dma' (copy engines)")
        self.mode = mode
        self.pg = process_group if process_group is not None else dist.group.WORLD
        self.n = dist.get_world_size(self.pg)
        self.rank = dist.get_rank(self.pg)
        if self.n > 8:
            raise ValueError("peer-memory update supports at most 8 ranks (one NVSwitch node)")
        self.max_slots = int(max_slots)
        self.flags = torch.zeros(2 * self.n * self.max_slots, dtype=torch.int64, device=G.device)
        self.step_dev = torch.zeros(1, dtype=torch.int64, device=G.device)   # this rank's step number
        self.G, self.W = G, W
        # dma: lane src of R receives rank src's gradient for this rank's parts
        self._lane = -(-G.numel() // 4) * 4 * G.element_size()     # 16-byte aligned lanes
        self.R = (torch.empty(self.n * self._lane // G.element_size(), dtype=G.dtype, device=G.device)
                  if mode == "dma" else None)
        bufs = (G, W, self.flags) + ((self.R,) if self.R is not None else ())
        try:
            mine = [self._handle(t) for t in bufs]
        except RuntimeError as e:
            mine = str(e)
        allh = [None] * self.n
        dist.all_gather_object(allh, mine, group=self.pg)
        bad = [h for h in allh if isinstance(h, str)]
        if bad:
            raise RuntimeError("IPC handles unavailable: " + "; ".join(bad))
        self._opened: dict = {}
        ptrs, err = [], ""
        try:
            for p in range(self.n):
                if p == self.rank:
                    ptrs.append([t.data_ptr() for t in bufs])
                else:
                    ptrs.append([self._open(p, h, off) for h, off in allh[p]])
        except RuntimeError as e:
            err = str(e)
        errs = [None] * self.n                      # all ranks agree: every mapping or none
        dist.all_gather_object(errs, err, group=self.pg)
        if any(errs):
            self.close()
            raise RuntimeError("peer mapping failed: " + "; ".join(e for e in errs if e))
        self.g_ptrs = (ctypes.c_void_p * self.n)(*[ptrs[p][0] for p in range(self.n)])
        self.w_ptrs = (ctypes.c_void_p * self.n)(*[ptrs[p][1] for p in range(self.n)])
        self.f_ptrs = (ctypes.c_void_p * self.n)(*[ptrs[p][2] for p in range(self.n)])
        if mode == "dma":
            self.r_ptrs = [ptrs[p][3] for p in range(self.n)]
            lane = self._lane
            self.g_lanes = (ctypes.c_void_p * self.n)(*[
                G.data_ptr() if s == self.rank else self.R.data_ptr() + s * lane for s in range(self.n)])
            self.w_local = (ctypes.c_void_p * self.n)(*[
                W.data_ptr() if p == self.rank else None for p in range(self.n)])
        self._sp = ctypes.c_void_p(self.step_dev.data_ptr())
        self.step_no = 0
        self.slot = 0
        self.parts: list[tuple[int, int]] = []      # this rank's [lo, hi) per slot
        dist.barrier(group=self.pg)

    @staticmethod
    def _handle(t: torch.Tensor):
        buf = ctypes.create_string_buffer(64)
        off = ctypes.c_longlong()
        _abi.call("omni_ipc_handle", ctypes.c_void_p(t.data_ptr()), buf, ctypes.byref(off))
        return buf.raw, off.value

    def _open(self, peer: int, h: bytes, off: int) -> int:
        key = (peer, h)
        if key not in self._opened:                 # one mapping per peer allocation
            base = ctypes.c_void_p()
            _abi.call("omni_ipc_open", h, ctypes.byref(base))
            self._opened[key] = base.value
        return self._opened[key] + off

    def part(self, lo: int, hi: int) -> tuple[int, int]:
        return owned_part(lo, hi, self.n, self.rank)

    def begin_step(self, stream=None) -> None:
        s = stream if stream is not None else torch.cuda.current_stream(self.G.device)
        _abi.call("omni_p2p_step", self._sp, ctypes.c_void_p(s.cuda_stream))
        self.step_no += 1
        self.slot = 0

    def layer(self, lo: int, hi: int, V: torch.Tensor, w_read: torch.Tensor, eta: float, mu: float,
              lam: float, stream=None) -> None:
        """Enqueue (on ``stream``) this rank's part of the fused update of
        W[lo:hi].  ``eta``/``lam`` already carry the mean's 1/N."""
        if self.slot >= self.max_slots:
            raise ValueError("more layer slices than max_slots")
        s = ctypes.c_void_p((stream if stream is not None
                             else torch.cuda.current_stream(self.G.device)).cuda_stream)
        slot = self.slot
        self.slot += 1
        esz = self.G.element_size()
        if self.mode == "dma":                   # push my gradient parts into the owners' lanes
            lane = self._lane
            for p in range(self.n):
                if p == self.rank:
                    continue
                a, b = owned_part(lo, hi, self.n, p)
                _abi.call("omni_copy_async", ctypes.c_void_p(self.r_ptrs[p] + self.rank * lane + a * esz),
                          ctypes.c_void_p(self.G.data_ptr() + a * esz), (b - a) * esz, s)
        _abi.call("omni_p2p_signal", self.f_ptrs, self.n, self.rank, self.GRAD_READY, slot,
                  self.max_slots, self._sp, s)
        _abi.call("omni_p2p_wait", ctypes.c_void_p(self.flags.data_ptr()), self.n, self.rank,
                  self.GRAD_READY, slot, slot + 1, self.max_slots, self._sp, s)
        a, b = self.part(lo, hi)
        dma = self.mode == "dma"
        if b > a:
            _abi.call("omni_p2p_reduce_sgd_f32", self.g_lanes if dma else self.g_ptrs,
                      self.w_local if dma else self.w_ptrs, self.n, self.rank, a, b,
                      ctypes.c_void_p(V.data_ptr()), ctypes.c_void_p(w_read.data_ptr()),
                      float(eta), float(mu), float(lam), s)
        if dma and b > a:                        # send my part of W to every peer
            for p in range(self.n):
                if p != self.rank:
                    _abi.call("omni_copy_async", ctypes.c_void_p(self.w_ptrs[p] + a * esz),
                              ctypes.c_void_p(self.W.data_ptr() + a * esz), (b - a) * esz, s)
        _abi.call("omni_p2p_signal", self.f_ptrs, self.n, self.rank, self.W_DONE, slot,
                  self.max_slots, self._sp, s)
        if len(self.parts) <= slot:
            self.parts.append((lo, hi))

    def finish(self, stream=None) -> None:
        """Block ``stream`` until every rank's W writes of this step landed here."""
        s = stream if stream is not None else torch.cuda.current_stream(self.G.device)
        _abi.call("omni_p2p_wait", ctypes.c_void_p(self.flags.data_ptr()), self.n, self.rank,
                  self.W_DONE, 0, self.slot, self.max_slots, self._sp,
                  ctypes.c_void_p(s.cuda_stream))

    def gather_momentum(self, V: torch.Tensor) -> None:
        """Make V complete on every rank (each rank holds only its parts):
        zero the other ranks' parts, then a sum allreduce (exact: x + 0)."""
        import torch.distributed as dist

        keep = torch.zeros_like(V, dtype=torch.bool)
        for lo, hi in self.parts:
            a, b = self.part(lo, hi)
            keep[a:b] = True
        V.masked_fill_(~keep, 0.0)
        dist.all_reduce(V, group=self.pg)

    def close(self) -> None:
        for base in self._opened.values():
            _abi.call("omni_ipc_close", ctypes.c_void_p(base))
        self._opened.clear()


class _Done:
    """Completion handle of an allreduce issued on a communicator stream:
    ``wait()`` makes the caller's current stream wait for it (no host block)."""

    def __init__(self, stream):
        self._ev = torch.cuda.Event()
        self._ev.record(stream)

    def wait(self) -> None:
        torch.cuda.current_stream().wait_event(self._ev)


class SessionComm:
    """The data-parallel session's collectives on the library's own NCCL
    communicator (C-ABI), one per process group: torch.distributed only
    bootstraps it (the unique id) and names the ranks.

    * ``allreduce_async(t)``: issued on a dedicated communicator stream after
      the work already queued on the caller's stream (a layer's weight
      gradient), so it overlaps the rest of the backward; returns a handle
      whose ``wait()`` orders the caller's stream after it;
    * ``gather_to_root`` / ``scatter_from_root`` / ``broadcast``: the merged-FC
      exchanges (pool5 activations and labels to rank 0, their gradients
      back), as grouped point-to-point calls on the caller's stream."""

    def __init__(self, process_group, device: torch.device):
        import torch.distributed as dist

        self.pg = process_group
        self.rank = dist.get_rank(process_group)
        self.world = dist.get_world_size(process_group)
        uid = [unique_id() if self.rank == 0 else None]
        root = dist.get_global_rank(process_group, 0) if process_group is not dist.group.WORLD else 0
        dist.broadcast_object_list(uid, src=root, group=process_group)
        self.comm = Communicator.init_rank(self.world, uid[0], self.rank, device.index)
        self.stream = torch.cuda.Stream(device=device)

    def allreduce_async(self, t: torch.Tensor) -> "_Done":
        cur = torch.cuda.current_stream(t.device)
        self.stream.wait_stream(cur)
        self.comm.allreduce_sum(t, stream=self.stream)
        return _Done(self.stream)

    def allreduce(self, t: torch.Tensor) -> torch.Tensor:
        return self.comm.allreduce_sum(t)

    def broadcast(self, t: torch.Tensor, root: int = 0) -> torch.Tensor:
        return self.comm.broadcast(_f32(t), root) if t.dtype == torch.float32 else self._bcast_bits(t, root)

    def _bcast_bits(self, t, root):
        self.comm.broadcast(t.view(torch.float32), root)
        return t

    def gather_to_root(self, src: torch.Tensor, dst_parts: list | None) -> None:
        """Rank r's ``src`` -> ``dst_parts[r]`` on rank 0 (int32 moves as its bits)."""
        with group():
            if self.rank == 0:
                for r in range(self.world):
                    if r == 0:
                        dst_parts[0].copy_(src)
                    else:
                        self.comm.recv(_f32(dst_parts[r]), r)
            else:
                self.comm.send(_f32(src), 0)

    def scatter_from_root(self, dst: torch.Tensor, src_parts: list | None) -> None:
        with group():
            if self.rank == 0:
                for r in range(self.world):
                    if r == 0:
                        dst.copy_(src_parts[0])
                    else:
                        self.comm.send(_f32(src_parts[r]), r)
            else:
                self.comm.recv(_f32(dst), 0)

    def close(self) -> None:
        self.comm.destroy()


class GroupExchange:
    """The collectives of groups.GroupRuntime on the library's own NCCL
    communicators (C-ABI): the world communicator, its split into the g
    compute groups (color = group, key = member) and into the k cross-group
    sets (color = member, key = group).  torch.distributed only bootstraps
    the unique id.  Calls run on the caller's (torch current) stream except
    ``all_to_all_async``, which runs on a dedicated stream ordered after the
    caller's work and returns a handle whose ``wait()`` orders the caller
    after it (the per-layer exchanges overlapping the backward)."""

    def __init__(self, plan, device: torch.device):
        import torch.distributed as dist

        self.rank = dist.get_rank()
        uid = [unique_id() if self.rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        self.world = Communicator.init_rank(plan.N, uid[0], self.rank, device.index)
        self.group = self.world.split(plan.group_of(self.rank), plan.member_of(self.rank))
        self.cross = self.world.split(plan.member_of(self.rank), plan.group_of(self.rank))
        self.stream = torch.cuda.Stream(device=device)

    def group_allreduce(self, t: torch.Tensor) -> None:
        self.group.allreduce_sum(t)

    def cross_allgather(self, t: torch.Tensor, out: torch.Tensor) -> None:
        """out row i = group i's t (this rank's member index in every group)."""
        self.cross.allgather(t, out)

    def world_allreduce(self, t: torch.Tensor) -> None:
        self.world.allreduce_sum(t)

    def world_allgather(self, t: torch.Tensor, out: torch.Tensor) -> None:
        self.world.allgather(t, out)

    def all_to_all(self, parts: list, recv: torch.Tensor) -> None:
        self.world.all_to_all(parts, recv)

    def all_to_all_async(self, parts: list, recv: torch.Tensor) -> "_Done":
        self.stream.wait_stream(torch.cuda.current_stream(recv.device))
        self.world.all_to_all(parts, recv, stream=self.stream)
        return _Done(self.stream)

    def close(self) -> None:
        for c in (self.cross, self.group, self.world):
            c.destroy()


def _f32(t: torch.Tensor) -> torch.Tensor:
    """A contiguous float32 view of the same bytes (int32 labels travel as bits)."""
    if t.dtype == torch.float32:
        return t
    if t.element_size() != 4:
        raise ValueError("only 4-byte element types travel through the float32 communicator calls")
    return t.view(torch.float32)
