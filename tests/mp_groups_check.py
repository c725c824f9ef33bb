"""Multi-GPU check of the compute-group runtime (NCCL, one process per GPU).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/mp_groups_check.py --g G

Runs GroupRuntime with the CUDA backend (3xTF32) on the reference TinyCNN and
compares the final master model and event log with the float64 oracle's
deterministic simulate (rank 0 prints one JSON line).
"""

import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import refcnn as R  # noqa: E402
from paper_1606_04487_b200.cluster import ExecutionPlan  # noqa: E402
from paper_1606_04487_b200.groups import CudaBackend, GroupRuntime  # noqa: E402
from paper_1606_04487_b200.problems import TinyCNNProblem  # noqa: E402
from paper_1606_04487_b200.sgd import Hyperparams  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--g", type=int, default=2)
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--overlap", action="store_true", help="layer-aligned shards, per-layer exchange")
    ap.add_argument("--p2p", action="store_true", help="exchanges over NVLink peer memory (DMA)")
    ap.add_argument("--replicated", action="store_true", help="unsharded: every rank holds W, V, snapshots")
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    world = dist.get_world_size()
    plan = ExecutionPlan(world, args.g)
    hp = Hyperparams(eta=0.05, mu=0.9, lam=1e-3, b=16)
    prob = TinyCNNProblem(8, 4, seed=3, n_examples=64, precision="3xtf32", device=dev)
    W0 = torch.from_numpy(prob.initial_weights().astype(np.float32)).to(dev)
    rt = GroupRuntime(plan, CudaBackend(prob, hp.b // plan.k), hp, W0, prob.n_examples, seed=11,
                      overlap=args.overlap, p2p=args.p2p,
                      sharded=not args.replicated)
    rt.run(args.rounds)
    torch.cuda.synchronize()
    W_master = rt.W                      # (sharded runtime: a collective, every rank)
    if dist.get_rank() == 0:
        layers = R.tiny_cnn_layers(8, 4)

        def grad_fn(W, batch):
            return R.grad(layers, 1, 8, W, *batch)

        def sample_fn(rng, b):
            idx = rng.integers(0, 64, size=b)
            return prob.images[idx], prob.labels[idx]

        Wr, _, ev = R.simulate(grad_fn, sample_fn, prob.initial_weights(), args.g, 4.0, 0.5, hp.eta,
                               hp.mu, hp.lam, hp.b, args.rounds * args.g, seed=11)
        got = W_master.double().cpu().numpy()
        err = float(np.linalg.norm(got - Wr) / np.linalg.norm(Wr))
        ev_ok = [(e.group_id, e.read_step, e.write_step, e.staleness) for e in rt.events] == \
                [tuple(e[:4]) for e in ev]
        print(json.dumps({"world": world, "g": args.g, "k": plan.k, "updates": rt.t,
                          "weights_rel_err": err, "events_match": ev_ok, "pass": ev_ok and err < 1e-4}))
    rt.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
