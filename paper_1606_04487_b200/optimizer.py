"""Algorithm 1: the asynchrony-aware optimizer (SPEC.md
module auto-optimizer, §5 / Appendix E.3-E.4).

The paper's optimizer sits on top of the training step: it picks the number
of compute groups g, the momentum mu and the step size eta by short probes,
starting from the most asynchronous configuration that saturates the server
and halving g while the best explicit momentum is 0 (asynchrony already
supplies all the momentum the problem wants).  The reference ships only the
specification; this module implements it over the simulator
(``simulator.simulate`` -- device-resident for GPU problems), in simulated
seconds, so a probe costs the same number of *updates* the real cluster would
do in that time (the HE model decides how fast each g is).

SPEC decisions followed: probe and epoch budgets are simulated seconds;
probes are paired (same start state, same batch-stream seed); losses are
compared on the trailing-50 mean; ties after 5 extension rounds go to
(lower eta, then lower mu); the cold-start sync sweep fixes mu = 0.9.
"""

from __future__ import annotations

import csv
import json
from dataclasses import dataclass, field, replace
from typing import Optional, Sequence

import numpy as np

from .cluster import ExecutionPlan, PhaseProfile, min_saturating_groups, power_of_two_divisors
from .sgd import Hyperparams, SGDState, child_seed

TRAILING = 50
MAX_EXTENSIONS = 5
SYNC_ETAS = (0.1, 0.01, 0.001, 0.0001, 0.00001)


@dataclass(frozen=True)
class GridSpec:
    momentum_grid: tuple = (0.0, 0.3, 0.6, 0.9)
    probe_budget: float = 30.0        # simulated seconds per grid point
    winner_threshold: float = 0.05    # relative trailing-loss gap that makes a clear winner
    group_candidates: Optional[tuple] = None

    def __post_init__(self) -> None:
        if not self.momentum_grid:
            raise ValueError("momentum grid is empty")
        if self.probe_budget <= 0:
            raise ValueError("probe_budget must be positive")
        if self.winner_threshold < 0:
            raise ValueError("winner_threshold must be >= 0")


@dataclass(frozen=True)
class EpochConfig:
    T: float = 600.0                  # simulated seconds of training per epoch
    target_loss: Optional[float] = None
    max_epochs: int = 5

    def __post_init__(self) -> None:
        if self.T <= 0 or self.max_epochs < 1:
            raise ValueError("T must be positive and max_epochs >= 1")


@dataclass(frozen=True)
class ProbeResult:
    state: SGDState
    loss: float          # trailing-50 mean of the sampled loss
    diverged: bool
    updates: int


@dataclass(frozen=True)
class DecisionRecord:
    epoch: int
    g: int
    mu: float
    eta: float
    probe_overhead_frac: float
    end_loss: float
    checkpoint: str


@dataclass
class DecisionLog:
    records: list = field(default_factory=list)

    def write_csv(self, path) -> None:
        with open(path, "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["epoch", "g", "mu", "eta", "probe_overhead_frac", "end_loss", "checkpoint"])
            for r in self.records:
                w.writerow([r.epoch, r.g, r.mu, r.eta, f"{r.probe_overhead_frac:.6f}",
                            repr(r.end_loss), r.checkpoint])


class SimEnv:
    """The simulation environment probes run in: a problem, N devices, a
    PhaseProfile (measured on B200 or synthetic), the group batch and the
    batch-stream seed.  Probes of one search round are paired (same start
    state, same seed); every training epoch advances ``seed_cursor`` so
    successive epochs draw fresh batches (the cursor is what a checkpoint
    records as ``seed_cursor`` to resume the same batch sequence)."""

    def __init__(self, problem, N: int, profile: PhaseProfile, b: int, seed: int = 0,
                 service_mode: str = "deterministic", loss_sample_interval: int = 1):
        self.problem, self.N, self.profile, self.b = problem, N, profile, b
        self.seed, self.service_mode, self.loss_sample_interval = seed, service_mode, loss_sample_interval
        self.sim_seconds = 0.0        # everything probed or trained, charged to the budget
        self.seed_cursor = 0          # training epochs run so far

    def current_seed(self) -> int:
        """Batch-stream seed of the current round: child_seed(seed, 4, cursor)
        (sgd.py:43-46 derivation), the plain seed before the first epoch."""
        return self.seed if self.seed_cursor == 0 else child_seed(self.seed, 4, self.seed_cursor)

    def run(self, state: SGDState, g: int, mu: float, eta: float, sim_seconds: float,
            train: bool = False) -> ProbeResult:
        from .simulator import SimConfig, simulate

        cfg = SimConfig(plan=ExecutionPlan(self.N, g), profile=self.profile,
                        hp=Hyperparams(eta=eta, mu=mu, b=self.b), problem=self.problem,
                        service_mode=self.service_mode, max_sim_seconds=sim_seconds,
                        seed=self.current_seed(), init=state,
                        loss_sample_interval=self.loss_sample_interval)
        tr = simulate(cfg)
        self.sim_seconds += sim_seconds
        if train:
            self.seed_cursor += 1
        losses = np.asarray(tr.loss_values, dtype=np.float64)
        tail = losses[-TRAILING:] if losses.size else np.array([np.inf])
        loss = float(np.mean(tail)) if not tr.diverged else float("inf")
        return ProbeResult(tr.final_state, loss, tr.diverged, len(tr.events))


def _pick(results: dict, threshold: float):
    """Best (mu, eta) by trailing loss; the set still within `threshold` of it."""
    finite = {k: r for k, r in results.items() if not r.diverged and np.isfinite(r.loss)}
    if not finite:
        return None, []
    best_loss = min(r.loss for r in finite.values())
    tol = threshold * max(abs(best_loss), 1e-12)
    close = sorted(k for k, r in finite.items() if r.loss <= best_loss + tol)
    best = min(finite, key=lambda k: (finite[k].loss, k[1], k[0]))
    return best, close


def grid_search(grid: GridSpec, state: SGDState, g: int, env, etas: Sequence[float],
                last: Optional[tuple] = None) -> tuple:
    """Algorithm 1's gridSearch(M, H | W, g): every (mu, eta) probed for
    probe_budget simulated seconds from the same state and seed; returns the
    lowest trailing loss.  If the runner-up is within winner_threshold, the
    survivors are extended by another probe_budget (up to 5 times; remaining
    ties go to lower eta, then lower mu).  Pruning (Appendix E.3): when eta
    equals the last eta*, momenta above the last mu* are skipped."""
    points = []
    for eta in etas:
        for mu in grid.momentum_grid:
            if last is not None and eta == last[1] and mu > last[0]:
                continue
            points.append((mu, eta))
    if not points:
        raise ValueError("grid search has no points after pruning")
    budget = grid.probe_budget
    results = {p: env.run(state, g, p[0], p[1], budget) for p in points}
    best, close = _pick(results, grid.winner_threshold)
    if best is None:
        raise RuntimeError(f"grid search at g={g}: every configuration diverged "
                           f"(points {points}, probe {budget} sim-s)")
    for _ in range(MAX_EXTENSIONS):
        if len(close) <= 1:
            break
        budget += grid.probe_budget           # survivors run again for the longer budget
        results = {p: env.run(state, g, p[0], p[1], budget) for p in close}
        best, close = _pick(results, grid.winner_threshold)
        if best is None:
            raise RuntimeError(f"grid search at g={g}: all survivors diverged on extension")
    if len(close) > 1:                        # stability-preferring tie break
        best = min(close, key=lambda k: (k[1], k[0]))
    return best


def refine_zero_momentum(grid: GridSpec, state: SGDState, g: int, env, eta: float) -> float:
    """Appendix E.3: after mu* = 0, also try mu = 0.1 and 0.2; best of {0, 0.1, 0.2}."""
    g2 = replace(grid, momentum_grid=(0.0, 0.1, 0.2))
    mu, _ = grid_search(g2, state, g, env, [eta])
    return mu


def init_groups(N: int, profile: PhaseProfile, candidates: Optional[Sequence[int]] = None):
    """Smallest g that saturates the server (§5.2), via the cluster model."""
    return min_saturating_groups(N, profile, candidates)


def cold_start(problem, env, grid: GridSpec, state: Optional[SGDState] = None):
    """Appendix E.4: (1) synchronous sweep with mu = 0.9 over eta in
    {1e-1 .. 1e-5}, stopping when the loss worsens; (2) for g = 2, 4, ... up
    to the saturating count, a grid over mu x {eta*_last, eta*_last/10} with
    the pruning rule; (3) race the candidates probe by probe until one leads by
    winner_threshold; (4) train the winner for one probe budget.  Returns
    (g, mu, eta, warm state)."""
    state = state if state is not None else problem.initial_state()
    best_eta, best_loss = None, np.inf
    for eta in SYNC_ETAS:
        r = env.run(state, 1, 0.9, eta, grid.probe_budget)
        if r.diverged or not np.isfinite(r.loss):
            continue
        if best_eta is not None and r.loss > best_loss:
            break
        best_eta, best_loss = eta, r.loss
    if best_eta is None:
        raise RuntimeError("cold start: the synchronous sweep diverged for every step size")
    cands = {1: (0.9, best_eta)}
    cand_gs = list(grid.group_candidates or power_of_two_divisors(env.N))
    g_top = init_groups(env.N, env.profile, cand_gs).g
    last = (0.9, best_eta)
    g = 2
    while g <= g_top and g in cand_gs:
        try:
            last = grid_search(grid, state, g, env, [last[1], last[1] / 10], last=last)
            cands[g] = last
        except RuntimeError:
            break
        g *= 2
    # (3) race: every candidate extends probe by probe from the same state
    budget = grid.probe_budget
    winner = None
    for _ in range(MAX_EXTENSIONS):
        res = {g_: env.run(state, g_, mu, eta, budget) for g_, (mu, eta) in cands.items()}
        ok = {g_: r for g_, r in res.items() if not r.diverged and np.isfinite(r.loss)}
        if not ok:
            raise RuntimeError("cold start: every candidate diverged in the race")
        order = sorted(ok, key=lambda g_: ok[g_].loss)
        winner = order[0]
        if len(order) == 1 or ok[order[1]].loss - ok[winner].loss > grid.winner_threshold * abs(ok[winner].loss):
            break
        budget += grid.probe_budget
    mu, eta = cands[winner]
    warm = env.run(state, winner, mu, eta, grid.probe_budget).state
    return winner, mu, eta, warm


def optimize(problem, env, grid: GridSpec, epochs: EpochConfig, checkpoint_dir: Optional[str] = None,
             state: Optional[SGDState] = None, start: Optional[tuple] = None):
    """Algorithm 1: cold start (or ``start`` = (g, mu, eta, state)), then per
    epoch: grid search at the current g; while mu* = 0 (after
    refine_zero_momentum) and g > 1, halve g and search again; train
    (g, mu*, eta*) for T simulated seconds; checkpoint.  Probe time is charged
    to the budget and reported per epoch."""
    g, mu, eta, state = start if start is not None else cold_start(problem, env, grid, state)
    log = DecisionLog()
    for epoch in range(epochs.max_epochs):
        before = env.sim_seconds
        mu, eta = grid_search(grid, state, g, env, [eta, eta / 10], last=(mu, eta))
        if mu == 0.0:
            mu = refine_zero_momentum(grid, state, g, env, eta)
        while mu == 0.0 and g > 1:
            g //= 2
            mu, eta = grid_search(grid, state, g, env, [eta, eta / 10])
            if mu == 0.0:
                mu = refine_zero_momentum(grid, state, g, env, eta)
        probe = env.sim_seconds - before
        r = env.run(state, g, mu, eta, epochs.T, train=True)
        state = r.state
        ckpt = ""
        if checkpoint_dir is not None:
            import os

            # (g, mu, eta) of the epoch are in the decision log row that names the file
            ckpt = os.path.join(checkpoint_dir, f"epoch{epoch}.omnickpt")
            save_checkpoint(Checkpoint(W=np.asarray(state.W), V=np.asarray(state.V), t=state.t,
                                       seed_cursor=env.seed_cursor), ckpt)
        log.records.append(DecisionRecord(epoch, g, mu, eta, probe / (probe + epochs.T), r.loss, ckpt))
        if r.diverged or (epochs.target_loss is not None and r.loss <= epochs.target_loss):
            break
    return state, log


# ---------------------------------------------------------- checkpoints --
CKPT_MAGIC = "OMNISIM-CKPT"
CKPT_VERSION = "v1"


@dataclass
class Checkpoint:
    """text header ``OMNISIM-CKPT v1 dim=<d> t=<t> seed_cursor=<u64>``
    followed by d decimal values for W then d for V, newline-separated; each
    value is the shortest decimal that round-trips the binary64 exactly
    (Python's repr), so the format is lossless and human-inspectable."""

    W: np.ndarray
    V: np.ndarray
    t: int
    seed_cursor: int = 0


def save_checkpoint(ck: Checkpoint, path) -> None:
    W = np.asarray(ck.W, dtype=np.float64)
    V = np.asarray(ck.V, dtype=np.float64)
    if W.shape != V.shape or W.ndim != 1:
        raise ValueError("checkpoint W and V must be 1-D and the same length")
    if not (0 <= int(ck.seed_cursor) < 2 ** 64) or int(ck.t) < 0:
        raise ValueError("checkpoint t must be >= 0 and seed_cursor a u64")
    with open(path, "w") as f:
        f.write(f"{CKPT_MAGIC} {CKPT_VERSION} dim={W.shape[0]} t={int(ck.t)} seed_cursor={int(ck.seed_cursor)}\n")
        f.write("\n".join(map(repr, W.tolist())))
        f.write("\n")
        if V.size:
            f.write("\n".join(map(repr, V.tolist())))
            f.write("\n")


def load_checkpoint(path) -> Checkpoint:
    """Parse the SPEC format; a malformed header names the offending field."""
    with open(path) as f:
        header = f.readline().rstrip("\n").split(" ")
        body = f.read().split()
    if len(header) < 1 or header[0] != CKPT_MAGIC:
        raise ValueError(f"checkpoint header field 'magic': expected {CKPT_MAGIC!r}, got {header[:1]!r}")
    if len(header) < 2 or header[1] != CKPT_VERSION:
        got = header[1] if len(header) > 1 else None
        raise ValueError(f"checkpoint header field 'version': expected {CKPT_VERSION!r}, got {got!r}")
    fields = {}
    for tok in header[2:]:
        k, _, v = tok.partition("=")
        fields[k] = v
    vals = {}
    for key in ("dim", "t", "seed_cursor"):
        if key not in fields:
            raise ValueError(f"checkpoint header field {key!r}: missing")
        try:
            vals[key] = int(fields[key])
        except ValueError:
            raise ValueError(f"checkpoint header field {key!r}: not an integer ({fields[key]!r})") from None
    d = vals["dim"]
    if d < 0 or len(body) != 2 * d:
        raise ValueError(f"checkpoint header field 'dim': {d} does not match the {len(body)} values "
                         "(expected 2 x dim)")
    data = np.array([float(x) for x in body], dtype=np.float64)
    return Checkpoint(W=data[:d].copy(), V=data[d:].copy(), t=vals["t"], seed_cursor=vals["seed_cursor"])
