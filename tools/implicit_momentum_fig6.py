"""Theorem 1 / Fig. 6 on B200: implicit momentum induced by g asynchronous
groups (exponential service, explicit momentum 0), estimated with
estimate_implicit_momentum (simulator.py:244-321) on the TinyCNN problem.

    python tools/implicit_momentum_fig6.py [--runs 256] [--impl ours|reference] [--out f.json]

--impl reference runs the reference package (build container only: it needs
/root/reference) on the same configuration and seeds.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", type=int, default=256)
    ap.add_argument("--groups", default="1,2,4,8")
    ap.add_argument("--max-updates", type=int, default=150)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--eta", type=float, default=0.05)
    ap.add_argument("--n-examples", type=int, default=64)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    if a.impl == "reference":
        sys.path.insert(0, "/root/reference/pkg/src")
        import omnisim as M
        from omnisim.simulator import estimate_implicit_momentum
        prob = M.make_tiny_cnn(8, 4, seed=3, n_examples=a.n_examples)
    else:
        sys.path.insert(0, ROOT)
        import paper_1606_04487_b200 as M
        from paper_1606_04487_b200 import estimate_implicit_momentum
        from paper_1606_04487_b200.problems import TinyCNNProblem
        prob = TinyCNNProblem(8, 4, seed=3, n_examples=a.n_examples, precision="3xtf32")
    N = 8
    rows = []
    for g in (int(x) for x in a.groups.split(",")):
        cfg = M.SimConfig(plan=M.ExecutionPlan(N=N, g=g),
                          profile=M.PhaseProfile(T_cc=4.0, T_nc=0.0, t_fc=0.01),
                          hp=M.Hyperparams(eta=a.eta, mu=0.0, lam=0.0, b=8), problem=prob,
                          service_mode="exponential", max_updates=a.max_updates, seed=11)
        t0 = time.time()
        est = estimate_implicit_momentum(cfg, n_runs=a.runs)
        rows.append({"g": g, "theorem1_1_minus_1_over_g": 1.0 - 1.0 / g, "estimate": est,
                     "runs": a.runs, "seconds": time.time() - t0})
        print(json.dumps(rows[-1]), flush=True)
    out = {"impl": a.impl, "problem": f"TinyCNN s8c4 n_ex={a.n_examples} seed=3", "N": N,
           "profile": "T_cc=4, T_nc=0, t_fc=0.01 (conv-saturated: memoryless race)",
           "hp": f"eta={a.eta} mu=0 lam=0 b=8", "max_updates": a.max_updates, "seed": 11,
           "rows": rows}
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
