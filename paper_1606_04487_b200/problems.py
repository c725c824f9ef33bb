"""Drop-in CNN training problems (omnisim.problems, problems.py:152-279), on the GPU.

``CNNProblem`` implements the reference's ``TrainingProblem`` plug-in
(sgd.py:115-152) for any NetSpec: batches are sampled with replacement by the
caller's RNG exactly as the reference does (problems.py:197-199), gradients
use the mean-over-batch convention (:248), and every forward/backward runs on
the B200 through ``engine.GpuNet``.  At this boundary W and gradients are
float64 NumPy (as in the reference); ``device_session`` keeps the model in
HBM for the training loops.

``TinyCNNProblem`` is the reference's only CNN, with the same constructor,
validation, synthetic data and teacher labels (problems.py:168-199), so its
losses and gradients can be compared with the reference on identical inputs.
"""

from __future__ import annotations

import os
from typing import Any

import numpy as np
import torch

from . import kernels as K
from . import nets
from .engine import GpuNet
from .sgd import Hyperparams, SGDState, TrainingProblem
from .tensors import ConvSpec

HOST_DATA_LIMIT = 32 * 1024 * 1024  # elements; larger synthetic sets are generated on the device


def _rng(seed: int, *key: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence(seed, spawn_key=tuple(key)))


class Batch:
    """A sampled mini-batch: indices into the problem's dataset.  Unpacks to
    host (images, labels) arrays like the reference's batches."""

    __slots__ = ("idx", "_problem")

    def __init__(self, problem: "CNNProblem", idx: np.ndarray):
        self.idx = np.asarray(idx, dtype=np.int64)
        self._problem = problem

    def __len__(self) -> int:
        return 2

    def __iter__(self):
        p = self._problem
        if p.images is None:
            raise ValueError("this problem's dataset lives on the device only")
        yield p.images[self.idx]
        yield p.labels[self.idx]

    @property
    def size(self) -> int:
        return int(self.idx.size)


class HostBatch:
    """A batch already laid out for the device -- images NHWC float32, labels
    int32 -- in (preferably pinned) host memory; copied asynchronously on the
    compute stream when a step consumes it."""

    __slots__ = ("X", "y")

    def __init__(self, X: torch.Tensor, y: torch.Tensor):
        if X.dim() != 4 or X.dtype != torch.float32 or y.dtype != torch.int32:
            raise ValueError("HostBatch wants X (b, n, n, c) float32 and y (b,) int32")
        self.X, self.y = X, y

    @property
    def size(self) -> int:
        return int(self.X.shape[0])


class DeviceBatch:
    """Indices (int64, already on the device) into the problem's dataset."""

    __slots__ = ("idx",)

    def __init__(self, idx: torch.Tensor):
        self.idx = idx

    @property
    def size(self) -> int:
        return int(self.idx.numel())


class LossFuture:
    """A step's loss on its way to the host (DeviceSession.loss_future)."""

    def __init__(self, buf: torch.Tensor, event):
        self._buf, self._event = buf, event

    def result(self) -> float:
        self._event.synchronize()
        return float(self._buf[0])


class DeviceSession:
    """W, V resident in HBM; one step = batch load + forward + backward + K8.

    With ``process_group`` (a torch.distributed NCCL group; one process per
    GPU) the session is synchronous data parallel over that group: each rank
    steps on its own batch, every layer's gradient is allreduced as soon as
    the backward has produced it (async, overlapping the remaining backward),
    and the mean over ranks is folded into the fused update."""

    def __init__(self, problem: "CNNProblem", state: SGDState, hp: Hyperparams,
                 process_group=None, use_graph: bool = True, merged_fc: bool = False,
                 p2p: bool = False):
        self.problem = problem
        self.hp = hp
        dev = problem.device
        self.W = torch.from_numpy(np.ascontiguousarray(state.W, dtype=np.float32)).to(dev)
        self.V = torch.from_numpy(np.ascontiguousarray(state.V, dtype=np.float32)).to(dev)
        self.t = state.t
        self.engine = problem.engine(hp.b)
        self.pg = process_group
        # id(HostBatch) -> (slot, ready event, the batch itself): the entry is
        # only honoured for that very object (an id can be reused once the
        # batch is garbage collected); _slot_owner[s] is the staged batch that
        # slot s holds and no step has consumed yet
        self._staged: dict[int, tuple] = {}
        self._slot_owner = [None, None]
        self._slots = None
        self._slot_free = [None, None]
        self._next_slot = 0
        self._copy_stream = None
        # CUDA graph of a whole single-GPU step on device-resident batches:
        # captured on the second such step (the first eager one does all lazy
        # setup), replayed with the batch indices copied into a static buffer.
        self.use_graph = use_graph and not os.environ.get("OMNI_NO_GRAPH")
        self._graphs: dict = {}
        self._seen: dict = {}
        self._gidx = None
        self.world = 1
        self.rank = 0
        if process_group is not None:
            import torch.distributed as dist

            self.world = dist.get_world_size(process_group)
            self.rank = dist.get_rank(process_group)
        # Merged FC: rank 0 runs the fully connected layers for
        # the whole global batch on the gathered pool5 activations (FC model and
        # FC compute co-located, FC gradients never exchanged); the conv part is
        # data parallel and only the conv gradients are allreduced.
        self.merged_fc = bool(merged_fc)
        self.head = None
        if self.merged_fc:
            if process_group is None:
                raise ValueError("merged_fc needs a process group (data parallel)")
            head_spec, self.fc_off = nets.fc_head(problem.net)
            if self.rank == 0:
                f = self.engine.first_fc
                self.head = GpuNet(head_spec, self.world * hp.b, dev, problem.precision,
                                   input_grad=True, input_cs=self.engine.ops[f].inp.cs)

        # Peer-memory data parallelism: each layer's allreduce + update is one
        # kernel reading the peers' gradients over NVLink (comm.PeerUpdate).
        # (Mapped at the first step, and again if W is replaced.)
        self.p2p = None
        self.use_p2p = bool(p2p)
        if p2p and (process_group is None or self.merged_fc):
            raise ValueError("p2p needs a process group and excludes merged_fc")

    def _peer(self):
        """The peer-memory update for the current W, or None when the ranks
        cannot map each other's memory (then every rank uses NCCL allreduce)."""
        if self.p2p is None or self.p2p.W.data_ptr() != self.W.data_ptr():
            from .comm import PeerUpdate

            if self.p2p is not None:
                self.p2p.close()
            nslots = sum(1 for op in self.engine.ops if op.kind in ("conv", "fc"))
            try:
                self.p2p = PeerUpdate(self.engine.grad, self.W, nslots, self.pg,
                                      mode=os.environ.get("OMNI_P2P_MODE", "dma"))
            except RuntimeError as e:
                import warnings

                warnings.warn(f"peer-memory update unavailable ({e}); using NCCL allreduce")
                self.p2p, self.use_p2p = None, False
        return self.p2p

    def _comm(self):
        """The library's own NCCL communicator over the process group
        (comm.SessionComm; torch.distributed only bootstraps it)."""
        if getattr(self, "_scomm", None) is None:
            from .comm import SessionComm

            self._scomm = SessionComm(self.pg, self.problem.device)
        return self._scomm

    def _allreduce_hook(self, works):
        G = self.engine.grad
        sc = self._comm()

        def hook(lo, hi):
            w = sc.allreduce_async(G[lo:hi])
            works.append(w)
            return w

        return hook

    def prefetch(self, batch: "HostBatch") -> None:
        """Start the host->device copy of a future step's batch on a side stream
        (double-buffered), so it overlaps the current step's compute."""
        if not isinstance(batch, HostBatch):
            raise ValueError("prefetch takes a HostBatch")
        eng = self.engine
        if self._slots is None:
            self._copy_stream = torch.cuda.Stream(device=self.problem.device)
            self._slots = [(torch.empty_like(eng.input.value), torch.empty_like(eng.labels))
                           for _ in range(2)]
        slot = self._next_slot
        if self._slot_owner[slot] is not None:
            raise ValueError("prefetch: both staging slots hold prefetched batches that have not been "
                             "stepped yet (at most two outstanding prefetches)")
        self._next_slot ^= 1
        X, y = self._slots[slot]
        b = batch.size
        with torch.cuda.stream(self._copy_stream):
            if self._slot_free[slot] is not None:       # the step that read this slot is done
                self._copy_stream.wait_event(self._slot_free[slot])
            X[:b].copy_(batch.X, non_blocking=True)
            y[:b].copy_(batch.y, non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(self._copy_stream)
        self._staged[id(batch)] = (slot, ready, batch)
        self._slot_owner[slot] = batch

    # ------------------------------------------------------------ steps --
    def _compute_merged(self, wr: torch.Tensor, b: int) -> None:
        hp, eng = self.hp, self.engine
        sc = self._comm()
        f = eng.first_fc
        eng.forward(wr, b, stop=f)                          # conv part, data parallel
        act, dact = eng.ops[f].inp.value[:b], eng.ops[f].inp.grad[:b]
        labels = eng.labels[:b]
        head = self.head
        if self.rank == 0:
            gx = [head.input.value[r * b:(r + 1) * b] for r in range(self.world)]
            gy = [head.labels[r * b:(r + 1) * b] for r in range(self.world)]
        else:
            gx = gy = None
        sc.gather_to_root(act.contiguous(), gx)
        sc.gather_to_root(labels.contiguous(), gy)
        nb = self.world * b
        if self.rank == 0:                                  # FC head on the whole global batch
            Wfc = wr[self.fc_off:]
            if Wfc.data_ptr() % 16:                         # the head stages from 16-byte-aligned W
                if getattr(self, "_wfc", None) is None:
                    self._wfc = torch.empty_like(Wfc)
                self._wfc.copy_(Wfc)
                Wfc = self._wfc
            head.forward(Wfc, nb)
            head.backward(nb)
            sx = [head.input.grad[r * b:(r + 1) * b] for r in range(self.world)]
        else:
            sx = None
        sc.scatter_from_root(dact, sx)
        works = []

        def hook(lo, hi):   # conv gradients only; the head's 1/(N b) makes SUM the mean
            w = sc.allreduce_async(eng.grad[lo:hi])
            works.append(w)
            return w

        eng.backward(b, on_grad=hook, update=(self.W, self.V, wr, hp.eta, hp.mu, hp.lam), start=f)
        for w in works:
            w.wait()
        if self.rank == 0:
            K.sgd_momentum(self.W[self.fc_off:], self.V[self.fc_off:], head.grad, Wfc,
                           hp.eta, hp.mu, hp.lam)

    def _compute(self, wr: torch.Tensor, b: int) -> None:
        """forward + backward (+ overlapped allreduce) + fused update on the batch
        already in the engine's input buffers."""
        hp = self.hp
        if self.merged_fc:
            self._compute_merged(wr, b)
        elif self.use_p2p and self._peer() is not None:
            n, peer, V = self.world, self.p2p, self.V
            peer.begin_step()
            self.engine.forward(wr, b)
            self.engine.backward(b, update=(self.W, V, wr, hp.eta / n, hp.mu, hp.lam * n),
                                 fused_update=lambda lo, hi, s: peer.layer(
                                     lo, hi, V, wr, hp.eta / n, hp.mu, hp.lam * n, s))
            peer.finish()        # every rank's W writes of this step have landed here
        elif self.world > 1:
            # each layer's gradient is allreduced as soon as it exists and that
            # layer's update follows its allreduce (inside the backward)
            works = []
            n = self.world   # eta (G_sum/n + lam w) = (eta/n) (G_sum + n lam w)
            self.engine.forward(wr, b)
            self.engine.backward(b, on_grad=self._allreduce_hook(works),
                                 update=(self.W, self.V, wr, hp.eta / n, hp.mu, hp.lam * n))
            for w in works:
                w.wait()   # (already waited for by the updates; keeps the handles honest)
        else:   # the update runs layer by layer inside the backward
            self.engine.forward(wr, b)
            self.engine.backward(b, update=(self.W, self.V, wr, hp.eta, hp.mu, hp.lam))

    def _run_on_slot(self, slot: int, b: int, wr: torch.Tensor) -> None:
        eng = self.engine
        own = (eng.input.value, eng.labels)
        eng.input.value, eng.labels = self._slots[slot]   # consume the staged buffers in place
        eng._s2d_ready = 0                                # the input comes from the slot
        try:
            self._compute(wr, b)
        finally:
            eng.input.value, eng.labels = own            # launches already hold the pointers

    def _staged_entry(self, batch) -> bool:
        """Whether ``batch`` (this very object) sits prefetched in a slot."""
        e = self._staged.get(id(batch))
        if e is not None and e[2] is not batch:      # a recycled id: stale entry
            del self._staged[id(batch)]
            return False
        return e is not None

    def _graph_key(self, batch, w_read):
        if not (self.use_graph and (self.world == 1 or self.use_p2p) and w_read is None and
                self.engine.timer is None and self.engine.overlap):
            return None
        base = (self.W.data_ptr(), self.V.data_ptr())
        if isinstance(batch, DeviceBatch) and batch.size == self.engine.b:
            return ("device", self.problem.data.data_ptr()) + base
        if isinstance(batch, HostBatch) and batch.size == self.engine.b and self._staged_entry(batch):
            return ("host", self._staged[id(batch)][0]) + base
        return None

    def step(self, batch: Any, w_read: torch.Tensor | None = None) -> None:
        """V = mu V - eta (grad(w_read) + lam w_read); W += V, with w_read = W when
        synchronous (sgd.py:104-112).  Runs on the problem's device (its current
        stream), whichever device the caller has current."""
        with torch.cuda.device(self.problem.device):
            self._step(batch, w_read)

    def _step(self, batch: Any, w_read: torch.Tensor | None = None) -> None:
        """(step's body)

        Single-GPU steps on full device batches or prefetched host batches are
        captured in a CUDA graph on their second occurrence and replayed after."""
        wr = self.W if w_read is None else w_read
        key = self._graph_key(batch, w_read)
        staged = None
        if isinstance(batch, HostBatch) and self._staged_entry(batch):
            staged = self._staged.pop(id(batch))
            self._slot_owner[staged[0]] = None
        cur = torch.cuda.current_stream()
        if staged is not None:
            cur.wait_event(staged[1])                     # H2D of this batch done
        if key is not None and key in self._graphs:
            if key[0] == "device":
                self._gidx.copy_(batch.idx, non_blocking=True)
            self._graphs[key].replay()
        elif key is not None and self._seen.get(key, 0) >= 1:
            # second occurrence: capture (the first eager step did all lazy setup)
            g = torch.cuda.CUDAGraph()
            if key[0] == "device":
                if self._gidx is None or self._gidx.numel() != batch.size:
                    self._gidx = torch.empty_like(batch.idx)
                self._gidx.copy_(batch.idx)
                with torch.cuda.graph(g):
                    self.engine.prestage(wr)
                    self.engine.gather_batch(self.problem.data, self.problem.data_labels, self._gidx)
                    self._compute(wr, batch.size)
            else:
                with torch.cuda.graph(g):
                    self._run_on_slot(key[1], batch.size, wr)
            self._graphs[key] = g
            g.replay()                                     # capture does not execute
        else:
            if key is not None:
                self._seen[key] = self._seen.get(key, 0) + 1
            if staged is not None:
                self._run_on_slot(staged[0], batch.size, wr)
            else:
                self.engine.prestage(wr)          # weight layouts overlap the batch gather
                b = self.problem.load_batch(self.engine, batch)
                self._compute(wr, b)
        if staged is not None:
            free = torch.cuda.Event()
            free.record(cur)
            self._slot_free[staged[0]] = free
        self.t += 1

    def full_loss(self) -> float:
        return self.problem.full_loss_device(self.W)

    def last_loss(self) -> float:
        """Mean loss of the last step's batch (one 4-byte device-to-host read).
        Merged FC: the global-batch loss, computed on rank 0 and broadcast
        (a collective: every rank calls it)."""
        if self.merged_fc:
            buf = (self.head.loss_buf if self.rank == 0 else torch.zeros(1, device=self.W.device))
            self._comm().broadcast(buf, 0)
            return float(buf.item())
        return float(self.engine.loss_buf.item())

    def loss_future(self) -> "LossFuture":
        """Start the device-to-host copy of the last step's loss without
        blocking: ``.result()`` waits for that step only, so a caller that reads
        step i's loss after enqueuing step i+1 never drains the GPU pipeline."""
        # each future owns its pinned scalar (torch's caching host allocator)
        dst = torch.empty(1, dtype=torch.float32, pin_memory=True)
        dst.copy_(self.engine.loss_buf.view(-1)[:1], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        return LossFuture(dst, ev)

    def sync_fc(self) -> None:
        """Merged FC: copy rank 0's FC parameters and momentum to every rank
        (the other ranks never update them).  A collective."""
        if not self.merged_fc:
            return
        sc = self._comm()
        sc.broadcast(self.W[self.fc_off:], 0)
        sc.broadcast(self.V[self.fc_off:], 0)

    def sync_momentum(self) -> None:
        """Peer-memory mode: each rank holds V only for the parts it updates;
        make V complete on every rank (a collective)."""
        if self.p2p is not None:
            self.p2p.gather_momentum(self.V)

    def state(self) -> SGDState:
        self.sync_momentum()
        return SGDState(W=self.W.double().cpu().numpy(), V=self.V.double().cpu().numpy(), t=self.t)


class CNNProblem(TrainingProblem):
    """Softmax-CE training of a NetSpec on synthetic Gaussian images."""

    def __init__(self, net: nets.NetSpec | str, n_examples: int = 128, seed: int = 0,
                 labels: str | None = None, precision: str = "3xtf32", device=None):
        self.net = nets.get(net) if isinstance(net, str) else net
        if n_examples < 1:
            raise ValueError("n_examples must be >= 1")
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1606_04487_b200 needs a CUDA device (no CPU fallback)")
        self.seed = seed
        self.precision = precision
        self.device = torch.device(device if device is not None else "cuda")
        c, s, C = self.net.in_channels, self.net.in_size, self.net.classes
        per = c * s * s
        self._n = n_examples
        if labels is None:
            labels = "teacher" if per * C <= 4 * 1024 * 1024 else "uniform"
        if n_examples * per <= HOST_DATA_LIMIT:
            rng = _rng(seed, 0)
            images = rng.standard_normal((n_examples, c, s, s))
            if labels == "teacher":
                teacher = rng.standard_normal((C, per))
                lab = np.argmax(teacher @ images.reshape(n_examples, -1).T, axis=0)
            else:
                lab = rng.integers(0, C, size=n_examples)
            self.images, self.labels = images, lab
            self.data = torch.from_numpy(images.astype(np.float32)).to(self.device)
            self.data = self.data.permute(0, 2, 3, 1).contiguous()
            self.data_labels = torch.from_numpy(lab.astype(np.int32)).to(self.device)
        else:
            gen = torch.Generator(device=self.device)
            gen.manual_seed(seed)
            self.images = self.labels = None
            self.data = torch.randn((n_examples, s, s, c), generator=gen, device=self.device)
            self.data_labels = torch.randint(0, C, (n_examples,), generator=gen,
                                             device=self.device, dtype=torch.int32)
        self._engines: dict[int, GpuNet] = {}

    # ------------------------------------------------------------- API ---
    @property
    def dim(self) -> int:
        return self.net.dim

    @property
    def n_examples(self) -> int:
        return self._n

    def initial_weights(self) -> np.ndarray:
        """0.01 * N(0, 1) over the whole flat vector (problems.py:194-195)."""
        return 0.01 * _rng(self.seed, 1).standard_normal(self.dim)

    def sample_batch(self, rng: np.random.Generator, b: int) -> Batch:
        return Batch(self, rng.integers(0, self._n, size=b))

    def engine(self, b: int) -> GpuNet:
        e = self._engines.get(b)
        if e is None:
            e = GpuNet(self.net, b, self.device, self.precision)
            self._engines[b] = e
        return e

    def load_batch(self, engine: GpuNet, batch: Any) -> int:
        """Put a batch on the device (gather by index, or upload host arrays)."""
        if isinstance(batch, Batch):
            idx = torch.from_numpy(batch.idx).to(self.device, non_blocking=True)
            engine.gather_batch(self.data, self.data_labels, idx)
            return batch.size
        if isinstance(batch, DeviceBatch):
            engine.gather_batch(self.data, self.data_labels, batch.idx)
            return batch.size
        if isinstance(batch, HostBatch):
            b = batch.size
            engine.input.value[:b].copy_(batch.X, non_blocking=True)
            engine.labels[:b].copy_(batch.y, non_blocking=True)
            return b
        X, y = batch
        X = np.asarray(X)
        Xd = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32)).to(self.device)
        engine.load_batch(Xd.permute(0, 2, 3, 1), torch.from_numpy(np.asarray(y, dtype=np.int32)).to(self.device))
        return X.shape[0]

    def _w(self, W) -> torch.Tensor:
        if isinstance(W, torch.Tensor):
            return W
        W = np.asarray(W, dtype=np.float64)
        if W.shape != (self.dim,):
            raise ValueError(f"weight vector has shape {W.shape}, problem needs ({self.dim},)")
        return torch.from_numpy(W.astype(np.float32)).to(self.device)

    def _batch_size(self, batch) -> int:
        return batch.size if isinstance(batch, (Batch, HostBatch, DeviceBatch)) else len(batch[1])

    def loss(self, W, batch) -> float:
        with torch.cuda.device(self.device):
            return self._loss(W, batch)

    def _loss(self, W, batch) -> float:
        e = self.engine(self._batch_size(batch))
        b = self.load_batch(e, batch)
        return float(e.forward(self._w(W), b, need_grad=False).item())

    def grad(self, W, batch) -> np.ndarray:
        with torch.cuda.device(self.device):   # launches go to this problem's device / stream
            return self._grad(W, batch)

    def _grad(self, W, batch) -> np.ndarray:
        e = self.engine(self._batch_size(batch))
        b = self.load_batch(e, batch)
        _, G = e.loss_and_grad(self._w(W), b)
        return G.double().cpu().numpy()

    def full_loss_device(self, Wd: torch.Tensor, chunk: int = 256) -> float:
        with torch.cuda.device(self.device):
            return self._full_loss_device(Wd, chunk)

    def _full_loss_device(self, Wd: torch.Tensor, chunk: int = 256) -> float:
        n = self._n
        e = self.engine(min(n, chunk))
        tot = torch.zeros(1, dtype=torch.float64, device=self.device)
        for s0 in range(0, n, e.b):
            b = min(e.b, n - s0)
            idx = torch.arange(s0, s0 + b, device=self.device, dtype=torch.int64)
            e.gather_batch(self.data, self.data_labels, idx)
            tot += e.forward(Wd, b, need_grad=False).double() * b
        return float(tot.item() / n)

    def full_loss(self, W) -> float:
        return self.full_loss_device(self._w(W))

    def full_grad(self, W, chunk: int = 256) -> np.ndarray:
        return self.full_grad_device(self._w(W), chunk).cpu().numpy()

    def full_grad_device(self, Wd: torch.Tensor, chunk: int = 256) -> torch.Tensor:
        """Mean gradient over the whole dataset at device weights (float64, on device)."""
        with torch.cuda.device(self.device):
            return self._full_grad_device(Wd, chunk)

    def _full_grad_device(self, Wd: torch.Tensor, chunk: int = 256) -> torch.Tensor:
        n = self._n
        e = self.engine(min(n, chunk))
        acc = torch.zeros(self.dim, dtype=torch.float64, device=self.device)
        for s0 in range(0, n, e.b):
            b = min(e.b, n - s0)
            idx = torch.arange(s0, s0 + b, device=self.device, dtype=torch.int64)
            e.gather_batch(self.data, self.data_labels, idx)
            _, G = e.loss_and_grad(Wd, b)
            acc += G.double() * (b / n)
        return acc

    def device_session(self, state: SGDState, hp: Hyperparams, process_group=None,
                       use_graph: bool = True, merged_fc: bool = False,
                       p2p: bool = False) -> DeviceSession:
        return DeviceSession(self, state, hp, process_group, use_graph, merged_fc, p2p)


def make_cnn(net: str, n_examples: int = 128, seed: int = 0, **kw) -> CNNProblem:
    return CNNProblem(net, n_examples, seed, **kw)


class TinyCNNProblem(CNNProblem):
    """conv(3x3, 4 ch) -> ReLU -> 2x2 max-pool -> linear -> softmax-CE (problems.py:152-275)."""

    D_OUT = 4
    K = 3

    def __init__(self, image_size: int, classes: int, seed: int = 0, n_examples: int = 128,
                 precision: str = "3xtf32", device=None):
        if image_size < 4 or image_size > 16 or image_size % 2 != 0:
            raise ValueError("image_size must be even and in [4, 16]")
        if not 2 <= classes <= 10:
            raise ValueError("classes must be in [2, 10]")
        self.image_size = image_size
        self.classes = classes
        s = image_size
        self.spec = ConvSpec(n=s, k=self.K, d_in=1, d_out=self.D_OUT, stride=1, pad=1)
        self.feat = self.D_OUT * (s // 2) * (s // 2)
        self.k_size = self.D_OUT * self.K * self.K
        super().__init__(nets.tiny_cnn(s, classes), n_examples, seed, labels="teacher",
                         precision=precision, device=device)

    def predict_proba(self, W, X) -> np.ndarray:
        X = np.asarray(X)
        e = self.engine(X.shape[0])
        self.load_batch(e, (X, np.zeros(X.shape[0], dtype=np.int32)))
        e.forward(self._w(W), X.shape[0], need_grad=False)
        logits = e.logits.value[: X.shape[0], : self.classes].double()
        return torch.softmax(logits, dim=1).cpu().numpy()


def make_tiny_cnn(image_size: int, classes: int, seed: int = 0, n_examples: int = 128) -> TinyCNNProblem:
    return TinyCNNProblem(image_size, classes, seed, n_examples)
