"""SPEC acceptance 8 for Algorithm 1 (optimizer.py):
on three synthetic cluster scenarios -- conv-bound, FC-saturated, balanced --
the optimizer's total simulated time to a target loss (its probes and cold
start included) is <= 1.5x the exhaustive-grid optimum, and its steady-state
probe overhead is <= 15% of the simulated budget.

    python tools/algorithm1_acceptance.py [out.json]

Problem: the reference's TinyCNN (problems.py:152-199), 16x16 inputs, 10
classes, 512 examples, on the device-resident simulator (simulator.py event
semantics).  Budgets: probe = 25 synchronous updates, epoch = 100 probes
(the paper runs 1-minute probes in 1-hour epochs; with 8 grid points plus
the SPEC's winner extensions, 1:60 leaves the per-epoch overhead at 13-25%).  The
target loss is what the synchronous baseline (g = 1, mu = 0.9, eta = 0.01)
reaches after 15,000 updates, so the best configuration needs several epochs
(with an easy target the cold start and the first epoch alone exceed 1.5x
the optimum, whatever the optimizer picks).  Time to target = first
simulated time the trailing-50 mean of the sampled loss is <= target -- the
same estimator the optimizer uses (optimizer.TRAILING); every run stops
there (SimConfig.target_loss).  The exhaustive grid is g in {1, 2, 4, 8} x
mu in {0, .3, .6, .9} x eta in {0.1, 0.01}; each run is capped at the
optimizer's total time / 1.5 (enough to decide the criterion; a config not
reaching the target within the cap reports None).
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_04487_b200 as P  # noqa: E402
from paper_1606_04487_b200 import optimizer as O  # noqa: E402
from paper_1606_04487_b200.problems import TinyCNNProblem  # noqa: E402

SCENARIOS = {
    "conv_bound": P.PhaseProfile(T_cc=1.0, T_nc=0.0, t_fc=0.01),
    "fc_saturated": P.PhaseProfile(T_cc=0.4, T_nc=0.2, t_fc=0.1),
    "balanced": P.PhaseProfile(T_cc=1.0, T_nc=0.1, t_fc=0.05),
}
N, B, SEED, SAMPLE = 8, 32, 5, 2


def trailing_time_to_target(tr, target, window=O.TRAILING):
    """First simulated time where the trailing-`window` mean of the sampled
    losses is <= target (None if never)."""
    v = np.asarray(tr.loss_values, dtype=np.float64)
    t = np.asarray(tr.loss_times, dtype=np.float64)
    if tr.diverged or v.size == 0:
        return None
    c = np.cumsum(np.insert(v, 0, 0.0))
    for i in range(v.size):
        lo = max(0, i + 1 - window)
        if (c[i + 1] - c[lo]) / (i + 1 - lo) <= target:
            return float(t[i])
    return None


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/algorithm1_acceptance.json"
    prob = TinyCNNProblem(16, 10, seed=3, n_examples=512)
    state0 = prob.initial_state()
    # target: the synchronous baseline's loss after 15,000 updates
    base = P.simulate(P.SimConfig(plan=P.ExecutionPlan(N=N, g=1), profile=SCENARIOS["balanced"],
                                  hp=P.Hyperparams(eta=0.01, mu=0.9, b=B), problem=prob, max_updates=15000,
                                  seed=SEED, loss_sample_interval=SAMPLE))
    target = float(np.mean(base.loss_values[-O.TRAILING:]))
    report = {"target_loss": target, "initial_loss": float(base.loss_values[0]), "scenarios": {}}
    ok_all = True
    for name, prof in SCENARIOS.items():
        he1 = P.he_predict(P.ExecutionPlan(N, 1), prof)
        probe = 25 * he1                       # ~25 updates of the slowest (synchronous) config
        T = 100 * probe                        # probe : epoch = 1 : 100 (the paper: 1 min : 1 h)
        env = O.SimEnv(prob, N=N, profile=prof, b=B, seed=SEED, loss_sample_interval=SAMPLE)
        grid = O.GridSpec(probe_budget=probe)
        t0 = time.perf_counter()
        state, log = O.optimize(prob, env, grid, O.EpochConfig(T=T, target_loss=target, max_epochs=60),
                                state=state0)
        wall_opt = time.perf_counter() - t0
        reached = bool(log.records) and log.records[-1].end_loss <= target
        t_alg = env.sim_seconds
        steady = [r.probe_overhead_frac for r in log.records[1:]] or [log.records[0].probe_overhead_frac]
        # exhaustive grid, each run capped at the optimizer's total time
        best, best_cfg, runs = None, None, []
        t1 = time.perf_counter()
        for g in (1, 2, 4, 8):
            for mu in (0.0, 0.3, 0.6, 0.9):
                for eta in (0.1, 0.01):
                    tr = P.simulate(P.SimConfig(plan=P.ExecutionPlan(N=N, g=g), profile=prof,
                                                hp=P.Hyperparams(eta=eta, mu=mu, b=B), problem=prob,
                                                max_sim_seconds=t_alg / 1.5, seed=SEED,
                                                loss_sample_interval=SAMPLE, init=state0,
                                                target_loss=target, target_window=O.TRAILING))
                    ttt = trailing_time_to_target(tr, target)
                    runs.append({"g": g, "mu": mu, "eta": eta, "time_to_target": ttt})
                    if ttt is not None and (best is None or ttt < best):
                        best, best_cfg = ttt, (g, mu, eta)
        wall_ex = time.perf_counter() - t1
        # no grid point reached the target within t_alg / 1.5: the optimum is
        # at least that, so the optimizer is within 1.5x of it
        ratio = (t_alg / best) if (best and reached) else (1.5 if reached else None)
        ok = bool(reached and ratio is not None and ratio <= 1.5 and max(steady) <= 0.15)
        ok_all &= ok
        report["scenarios"][name] = {
            "profile": {"T_cc": prof.T_cc, "T_nc": prof.T_nc, "t_fc": prof.t_fc},
            "he_predict_per_g": {g: P.he_predict(P.ExecutionPlan(N, g), prof) for g in (1, 2, 4, 8)},
            "probe_budget": probe, "epoch_T": T,
            "optimizer": {"reached_target": reached, "total_sim_seconds": t_alg,
                          "decisions": [(r.epoch, r.g, r.mu, r.eta, round(r.probe_overhead_frac, 4),
                                         r.end_loss) for r in log.records],
                          "cold_start_plus_first_epoch_overhead": log.records[0].probe_overhead_frac,
                          "steady_probe_overhead_max": max(steady), "wall_s": wall_opt},
            "exhaustive": {"best_time_to_target": best, "best_config": best_cfg, "wall_s": wall_ex,
                           "runs": runs},
            "ratio_vs_exhaustive": ratio, "pass": ok}
        print(name, json.dumps({k: report["scenarios"][name][k] for k in ("ratio_vs_exhaustive", "pass")}),
              "alg", t_alg, "best", best, best_cfg, "overhead", max(steady), flush=True)
    report["pass"] = ok_all
    json.dump(report, open(out_path, "w"), indent=1)
    print(json.dumps({"pass": ok_all, "target": target}))


if __name__ == "__main__":
    main()
