"""Calibrate the Algorithm 1 acceptance scenarios: TinyCNN loss traces under
the simulator for a few (g, mu, eta) and profiles, to pick a target loss the
best configuration reaches in a few hundred updates.

    python tools/algorithm1_calibrate.py
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_04487_b200 as P  # noqa: E402
from paper_1606_04487_b200.problems import TinyCNNProblem  # noqa: E402


def main():
    prob = TinyCNNProblem(8, 4, seed=3, n_examples=64)
    prof = P.PhaseProfile(T_cc=1.0, T_nc=0.05, t_fc=0.05)
    out = {}
    for g in (1, 4):
        for mu in (0.0, 0.9):
            for eta in (0.1, 0.01):
                cfg = P.SimConfig(plan=P.ExecutionPlan(N=8, g=g), profile=prof,
                                  hp=P.Hyperparams(eta=eta, mu=mu, b=16), problem=prob,
                                  max_updates=1500, seed=5, loss_sample_interval=25)
                t0 = time.perf_counter()
                tr = P.simulate(cfg)
                dt = time.perf_counter() - t0
                out[f"g{g}_mu{mu}_eta{eta}"] = {"wall_s": dt, "diverged": tr.diverged,
                                                 "loss": [round(float(x), 4) for x in tr.loss_values[::6]],
                                                 "t": [round(float(x), 2) for x in tr.loss_times[::6]]}
                print(g, mu, eta, f"{dt:.2f}s", out[f"g{g}_mu{mu}_eta{eta}"]["loss"], flush=True)
    json.dump(out, open("gpurun_out/a1_calibrate.json", "w"), indent=1)


if __name__ == "__main__":
    main()
