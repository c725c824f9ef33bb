"""Algorithm 1 on the device-resident simulator with the PhaseProfile measured
on B200 by tools/async_he.py (CaffeNet: T_cc 3.43 ms, T_nc 0.49 ms, t_fc
0.81 ms), N = 8; the training problem is the TinyCNN so that the many probes
stay cheap.  Writes the decision log and a JSON summary.

    python tools/algorithm1_demo.py --out gpurun_out/alg1.json
"""
import argparse
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_04487_b200 as P  # noqa: E402
from paper_1606_04487_b200 import optimizer as O  # noqa: E402
from paper_1606_04487_b200.problems import TinyCNNProblem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--probe", type=float, default=0.05, help="simulated seconds per probe")
    ap.add_argument("--epoch", type=float, default=0.5, help="simulated seconds per epoch")
    ap.add_argument("--epochs", type=int, default=3)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    prof = P.PhaseProfile(T_cc=3.43e-3, T_nc=0.49e-3, t_fc=0.81e-3)
    prob = TinyCNNProblem(8, 4, seed=3, n_examples=128)
    env = O.SimEnv(prob, N=8, profile=prof, b=16, seed=5, loss_sample_interval=4)
    t0 = time.time()
    ckdir = tempfile.mkdtemp()
    state, log = O.optimize(prob, env, O.GridSpec(probe_budget=a.probe),
                            O.EpochConfig(T=a.epoch, max_epochs=a.epochs), checkpoint_dir=ckdir)
    out = {
        "problem": "TinyCNN s8c4 n_ex=128, b=16", "N": 8,
        "profile_s": {"T_cc": prof.T_cc, "T_nc": prof.T_nc, "t_fc": prof.t_fc},
        "init_groups": list(O.init_groups(8, prof)),
        "he_predict_s_per_update": {g: P.he_predict(P.ExecutionPlan(8, g), prof) for g in (1, 2, 4, 8)},
        "probe_budget_sim_s": a.probe, "epoch_sim_s": a.epoch,
        "initial_loss": prob.full_loss(prob.initial_weights()),
        "decisions": [r.__dict__ | {"checkpoint": os.path.basename(r.checkpoint)} for r in log.records],
        "sim_seconds_total": env.sim_seconds, "wall_s": time.time() - t0,
    }
    print(json.dumps(out, indent=1))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
