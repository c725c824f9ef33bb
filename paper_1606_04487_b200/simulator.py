"""Drop-in for omnisim.simulator's hot-path part: the g-group asynchronous schedule.

``simulate`` keeps the reference's event semantics exactly (simulator.py:123-213):
g groups snapshot the master model, draw a batch from their own stream,
"compute" for t_conv(k), queue FIFO at one serial FC server, and on
completion apply one momentum update with the gradient evaluated at their
snapshot (the regulariser uses the snapshot too).  With a GPU problem the
master W, V and every snapshot stay in HBM and each update is one fused
forward/backward + K8 launch sequence; the event order is host logic and
deterministic per seed.  ``groups.py`` runs the same schedule across real
GPUs.
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass, replace
from typing import Optional

import numpy as np

from .cluster import ExecutionPlan, PhaseProfile, t_conv
from .sgd import (DIVERGENCE_FACTOR, Hyperparams, LossTrace, SGDState, TrainingProblem,
                  batch_stream, child_seed, service_stream, sgd_step)

DEFAULT_BURN_IN = 100


@dataclass(frozen=True)
class SimConfig:
    plan: ExecutionPlan
    profile: PhaseProfile
    hp: Hyperparams
    problem: TrainingProblem
    service_mode: str = "deterministic"
    max_updates: Optional[int] = None
    max_sim_seconds: Optional[float] = None
    seed: int = 0
    init: Optional[SGDState] = None
    loss_sample_interval: int = 1
    record_models: bool = False
    # (extension, not in the reference) stop once the mean of the last
    # `target_window` sampled losses is <= target_loss -- time-to-target sweeps
    target_loss: Optional[float] = None
    target_window: int = 50

    def __post_init__(self) -> None:
        if self.service_mode not in ("deterministic", "exponential"):
            raise ValueError(f"unknown service_mode {self.service_mode!r}")
        if self.max_updates is None and self.max_sim_seconds is None:
            raise ValueError("need max_updates and/or max_sim_seconds")
        if self.max_updates is not None and self.max_updates < 1:
            raise ValueError("max_updates must be >= 1")
        if self.loss_sample_interval < 1:
            raise ValueError("loss_sample_interval must be >= 1")


@dataclass(frozen=True, slots=True)
class SimEvent:
    group_id: int
    read_step: int
    write_step: int
    staleness: int
    start_time: float
    fc_enqueue_time: float
    finish_time: float


@dataclass
class SimTrace:
    events: list
    loss_steps: np.ndarray
    loss_times: np.ndarray
    loss_values: np.ndarray
    final_state: SGDState
    diverged: bool = False
    models: Optional[np.ndarray] = None

    @property
    def write_times(self) -> np.ndarray:
        return np.array([e.finish_time for e in self.events])

    def to_loss_trace(self) -> LossTrace:
        return LossTrace(steps=self.loss_steps, sim_times=self.loss_times, losses=self.loss_values,
                         final_state=self.final_state, diverged=self.diverged)

    def write_csv(self, path) -> None:
        sampled = dict(zip(self.loss_steps.tolist(), self.loss_values.tolist()))
        with open(path, "w") as f:
            f.write("write_step,group_id,read_step,staleness,start_s,finish_s,loss\n")
            last = sampled.get(0, float("nan"))
            for e in self.events:
                last = sampled.get(e.write_step, last)
                f.write(f"{e.write_step},{e.group_id},{e.read_step},{e.staleness},"
                        f"{e.start_time:.6f},{e.finish_time:.6f},{last!r}\n")


class _HostModel:
    """Master model for problems without a device session (host arrays)."""

    def __init__(self, problem, state, hp):
        self.problem, self.state, self.hp = problem, state, hp

    @property
    def t(self):
        return self.state.t

    def snapshot(self):
        return self.state.W.copy()

    def apply(self, snapshot, batch):
        g = self.problem.grad(snapshot, batch)
        self.state = sgd_step(self.state, self.hp, g, snapshot)

    def finite(self):
        return bool(np.all(np.isfinite(self.state.W)))

    def full_loss(self):
        return self.problem.full_loss(self.state.W)

    def model_copy(self):
        return self.state.W.copy()

    def final(self):
        return self.state


class _DeviceModel:
    """Master W, V and snapshots resident in HBM (CNNProblem)."""

    def __init__(self, problem, state, hp):
        import torch

        self.torch = torch
        self.s = problem.device_session(state, hp)

    @property
    def t(self):
        return self.s.t

    def snapshot(self):
        return self.s.W.clone()

    def apply(self, snapshot, batch):
        self.s.step(batch, w_read=snapshot)

    def finite(self):
        return bool(self.torch.isfinite(self.s.W).all().item())

    def full_loss(self):
        return self.s.full_loss()

    def model_copy(self):
        return self.s.W.double().cpu().numpy()

    def final(self):
        return self.s.state()


def simulate(cfg: SimConfig) -> SimTrace:
    """Run the event loop until the update or sim-time budget, or divergence."""
    return _simulate(cfg)


def _simulate(cfg: SimConfig, on_write=None) -> SimTrace:
    """simulate(), plus ``on_write(i, model)`` after the i-th master update
    (i = 0 for the initial model) -- how the implicit-momentum estimator
    records device-resident trajectories without host copies."""
    g = cfg.plan.g
    conv_mean = t_conv(cfg.plan.k, cfg.profile)
    fc_mean = cfg.profile.t_fc
    exponential = cfg.service_mode == "exponential"
    batch_rngs = [batch_stream(cfg.seed, i) for i in range(g)]
    svc_rngs = [service_stream(cfg.seed, i) for i in range(g)] if exponential else None

    state = cfg.init if cfg.init is not None else cfg.problem.initial_state()
    model = (_DeviceModel if hasattr(cfg.problem, "device_session") else _HostModel)(cfg.problem, state, cfg.hp)
    initial_loss = model.full_loss()
    bound = DIVERGENCE_FACTOR * max(abs(initial_loss), 1.0)
    events: list[SimEvent] = []
    loss_steps, loss_times, loss_values = [model.t], [0.0], [initial_loss]
    models = [model.model_copy()] if cfg.record_models else None
    diverged = not np.isfinite(initial_loss)
    t0 = model.t
    if on_write is not None:
        on_write(0, model)

    def draw(i):
        if exponential:
            r = svc_rngs[i]
            return r.exponential(conv_mean), r.exponential(fc_mean)
        return conv_mean, fc_mean

    heap: list = []
    seq = 0
    for i in range(g):
        cd, fs = draw(i)
        batch = cfg.problem.sample_batch(batch_rngs[i], cfg.hp.b)
        heapq.heappush(heap, (cd, seq, i, model.snapshot(), model.t, 0.0, batch, fs))
        seq += 1

    fc_free = 0.0
    while not diverged:
        if cfg.max_updates is not None and model.t - t0 >= cfg.max_updates:
            break
        conv_done, _, i, snap, read_step, read_time, batch, fs = heap[0]
        finish = max(fc_free, conv_done) + fs
        if cfg.max_sim_seconds is not None and finish > cfg.max_sim_seconds:
            break
        heapq.heappop(heap)
        fc_free = finish
        model.apply(snap, batch)
        t = model.t
        events.append(SimEvent(i, read_step, t, t - 1 - read_step, read_time, conv_done, finish))
        if models is not None:
            models.append(model.model_copy())
        if on_write is not None:
            on_write(t - t0, model)
        if not model.finite():
            diverged = True
        if (t - t0) % cfg.loss_sample_interval == 0 or diverged:
            loss = model.full_loss()
            loss_steps.append(t)
            loss_times.append(finish)
            loss_values.append(loss)
            if not np.isfinite(loss) or loss > bound:
                diverged = True
            elif cfg.target_loss is not None and \
                    float(np.mean(loss_values[-cfg.target_window:])) <= cfg.target_loss:
                break
        if diverged:
            break
        cd, nfs = draw(i)
        nb = cfg.problem.sample_batch(batch_rngs[i], cfg.hp.b)
        heapq.heappush(heap, (finish + cd, seq, i, model.snapshot(), t, finish, nb, nfs))
        seq += 1

    return SimTrace(events=events, loss_steps=np.array(loss_steps), loss_times=np.array(loss_times),
                    loss_values=np.array(loss_values), final_state=model.final(), diverged=diverged,
                    models=np.array(models) if models is not None else None)


def measured_he(trace: SimTrace, burn_in: int = DEFAULT_BURN_IN) -> float:
    """Mean inter-write interval after discarding the first burn_in events."""
    if len(trace.events) <= burn_in + 1:
        raise ValueError(
            f"trace has {len(trace.events)} events; need more than burn_in + 1 = {burn_in + 1}")
    return float(np.diff(trace.write_times[burn_in:]).mean())


@dataclass(frozen=True)
class StalenessStats:
    mean: float
    histogram: dict


def staleness_stats(trace: SimTrace, burn_in: int = 0) -> StalenessStats:
    s = np.array([e.staleness for e in trace.events[burn_in:]])
    if s.size == 0:
        raise ValueError("trace has no events past burn_in")
    v, c = np.unique(s, return_counts=True)
    return StalenessStats(mean=float(s.mean()), histogram={int(a): int(b) for a, b in zip(v, c)})


def _signal_window(mags: np.ndarray, burn_in: int, signal_floor: float, n_models: int) -> int:
    """End of the fit window (simulator.py:296-304): the first t >= burn_in + 20
    where the averaged increment drops below signal_floor x its early level."""
    if burn_in + 21 >= mags.shape[0]:
        raise ValueError("max_updates too small for the burn-in window")
    threshold = signal_floor * float(np.mean(mags[burn_in:burn_in + 10]))
    for t in range(burn_in + 20, n_models - 1):
        if mags[t] < threshold:
            return t
    return n_models - 1


def estimate_implicit_momentum(cfg: SimConfig, n_runs: int, burn_in: Optional[int] = None,
                               signal_floor: float = 0.02) -> float:
    """Regression estimate of the momentum asynchrony induces (simulator.py:244-321,
    Theorem 1): average the master trajectories of ``n_runs`` seeded runs
    (seed child_seed(cfg.seed, 3, r)), then least-squares fit
    V(t+1) ~ a V(t) - c grad(W(t)) over the window where the averaged signal is
    alive, pooling time steps and coordinates; returns ``a``.

    With a GPU problem every trajectory stays in HBM (written by the event
    loop's update hook), the runs are summed in float64 on the device, the
    full gradients along the mean path are device passes, and the two-column
    least squares is solved from its 2x2 normal equations in float64."""
    if cfg.hp.mu != 0.0:
        raise ValueError("implicit-momentum estimation requires explicit momentum 0")
    if cfg.service_mode != "exponential":
        raise ValueError("implicit-momentum estimation requires exponential service")
    if cfg.max_updates is None:
        raise ValueError("cfg.max_updates must be set")
    if burn_in is None:
        burn_in = 3 * cfg.plan.g + 10
    if not hasattr(cfg.problem, "device_session"):
        return _estimate_host(cfg, n_runs, burn_in, signal_floor)

    import torch

    prob = cfg.problem
    T = cfg.max_updates + 1
    total = None
    n_ok = 0
    for r in range(n_runs):
        run_cfg = replace(cfg, seed=child_seed(cfg.seed, 3, r), record_models=False)
        path = torch.empty((T, prob.dim), dtype=torch.float32, device=prob.device)
        written = [0]

        def on_write(i, model, path=path, written=written):
            path[i].copy_(model.s.W)
            written[0] = i + 1

        trace = _simulate(run_cfg, on_write)
        if trace.diverged or written[0] != T:
            continue
        if total is None:
            total = path.double()
        else:
            total.add_(path)
        n_ok += 1
    if total is None:
        raise ValueError("no usable runs (all diverged or cut short)")
    mean_path = total.div_(n_ok)
    V = mean_path[1:] - mean_path[:-1]
    mags = V.abs().amax(dim=1).cpu().numpy()
    t_end = _signal_window(mags, burn_in, signal_floor, T)
    # normal equations of [V(t-1), -grad(t)] beta = V(t), accumulated in float64
    a11 = a12 = a22 = b1 = b2 = torch.zeros((), dtype=torch.float64, device=prob.device)
    rows = 0
    for t in range(burn_in + 1, t_end):
        gr = prob.full_grad_device(mean_path[t].float())
        v, y = V[t - 1], V[t]
        a11 = a11 + v.dot(v)
        a12 = a12 - v.dot(gr)
        a22 = a22 + gr.dot(gr)
        b1 = b1 + v.dot(y)
        b2 = b2 - gr.dot(y)
        rows += prob.dim
    if rows == 0:
        raise ValueError("signal window is empty; lower burn_in or raise max_updates")
    if n_ok * rows < 1000:
        raise ValueError(f"insufficient samples: {n_ok * rows} pooled triples < 1000")
    A = torch.stack([torch.stack([a11, a12]), torch.stack([a12, a22])]).cpu().numpy()
    bvec = torch.stack([b1, b2]).cpu().numpy()
    beta, *_ = np.linalg.lstsq(A, bvec, rcond=None)
    return float(beta[0])


def _estimate_host(cfg: SimConfig, n_runs: int, burn_in: int, signal_floor: float) -> float:
    """The same estimator for host problems (recorded float64 trajectories)."""
    paths = []
    for r in range(n_runs):
        trace = simulate(replace(cfg, seed=child_seed(cfg.seed, 3, r), record_models=True))
        if trace.diverged or trace.models is None or trace.models.shape[0] != cfg.max_updates + 1:
            continue
        paths.append(trace.models)
    if not paths:
        raise ValueError("no usable runs (all diverged or cut short)")
    mean_path = np.mean(paths, axis=0)
    V = np.diff(mean_path, axis=0)
    mags = np.max(np.abs(V), axis=1)
    t_end = _signal_window(mags, burn_in, signal_floor, mean_path.shape[0])
    xs, ys = [], []
    for t in range(burn_in + 1, t_end):
        xs.append(np.column_stack([V[t - 1], -cfg.problem.full_grad(mean_path[t])]))
        ys.append(V[t])
    if not xs:
        raise ValueError("signal window is empty; lower burn_in or raise max_updates")
    X, y = np.concatenate(xs), np.concatenate(ys)
    if len(paths) * X.shape[0] < 1000:
        raise ValueError(f"insufficient samples: {len(paths) * X.shape[0]} pooled triples < 1000")
    beta, *_ = np.linalg.lstsq(X, y, rcond=None)
    return float(beta[0])
