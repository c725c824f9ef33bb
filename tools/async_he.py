"""Free-running asynchronous groups on B200s + HE-model validation
(SURVEY §8(f) #1).  Launch with one process per GPU; rank 0 is the server,
ranks 1..N the workers:

    torchrun --nproc-per-node P --master-addr 127.0.0.1 tools/async_he.py \
        --groups 1,2 --updates 60 --out gpurun_out/async.json

For every g dividing N = P - 1 it measures, on this box:
  * PhaseProfile: T_cc = one GPU's gradient time for the group batch (CUDA
    events), T_nc = one-way P2P time of the model (250 MB for CaffeNet),
    t_fc = the server's service time per update (apply + reply);
  * the asynchronous run: seconds per update (measured_he over the server's
    write times), staleness histogram, and the replay check (the update log
    re-applied in order on the server GPU must reproduce the final model:
    bit-exact for k = 1);
and reports cluster.he_predict(ExecutionPlan(N, g), profile) next to it.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1606_04487_b200 import async_groups as A  # noqa: E402
from paper_1606_04487_b200.cluster import ExecutionPlan, PhaseProfile, he_predict, t_conv  # noqa: E402
from paper_1606_04487_b200.groups import CudaBackend  # noqa: E402
from paper_1606_04487_b200.problems import CNNProblem  # noqa: E402
from paper_1606_04487_b200.sgd import Hyperparams  # noqa: E402


def event_ms(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="caffenet")
    ap.add_argument("--batch", type=int, default=240, help="group batch (divisible by every k)")
    ap.add_argument("--groups", default="")
    ap.add_argument("--updates", type=int, default=60)
    ap.add_argument("--n-examples", type=int, default=512)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    os.environ.setdefault("NCCL_NVLS_ENABLE", "0")
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    ngpu = torch.cuda.device_count()
    dev = torch.device("cuda", rank % ngpu)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    N = world - 1
    groups = [int(x) for x in a.groups.split(",")] if a.groups else [g for g in range(1, N + 1) if N % g == 0]
    prob = CNNProblem(a.net, n_examples=a.n_examples, seed=5, labels="uniform", precision="tf32",
                      device=dev)
    gen = torch.Generator(device=dev).manual_seed(7)
    W0 = 0.01 * torch.randn(prob.dim, generator=gen, device=dev)
    hp = Hyperparams(eta=0.01, mu=0.0, lam=5e-4, b=a.batch)

    # ---- PhaseProfile on this box
    prof = {}
    if rank == 1:
        be = CudaBackend(prob, a.batch)
        idx = np.arange(a.batch) % a.n_examples
        prof["T_cc"] = event_ms(lambda: be.grad(W0, idx)) / 1e3
    buf = torch.empty_like(W0)
    dist.barrier()
    if rank in (0, 1):                               # one-way model transfer, server <-> a worker
        torch.cuda.synchronize()
        for rep in range(4):
            t0 = time.perf_counter()
            if rank == 0:
                dist.send(W0, dst=1)
                dist.recv(buf, src=1)
            else:
                dist.recv(buf, src=0)
                dist.send(buf, dst=0)
            torch.cuda.synchronize()
            if rep:
                prof.setdefault("rt", []).append(time.perf_counter() - t0)
        prof["T_nc"] = float(np.median(prof.pop("rt"))) / 2
    if rank == 0:                                    # server service: update + reply copy
        be0 = CudaBackend(prob, a.batch)
        V = torch.zeros_like(W0)
        Wt = W0.clone()
        snap = W0.clone()
        svc = event_ms(lambda: (be0.sgd(Wt, V, buf, snap, hp), snap.copy_(Wt))) / 1e3
        prof["t_fc"] = svc + prof["T_nc"]           # + the model going back
    dist.barrier()
    allp = [None] * world
    dist.all_gather_object(allp, prof)
    profile = PhaseProfile(T_cc=allp[1]["T_cc"], T_nc=allp[0]["T_nc"], t_fc=allp[0]["t_fc"])

    rows = []
    for g in groups:
        plan = ExecutionPlan(N, g)
        dist.barrier()
        if rank == 0:
            res = A.run_server(plan, CudaBackend(prob, a.batch // plan.k), hp, W0, a.updates)
        else:
            A.run_worker(plan, CudaBackend(prob, a.batch // plan.k), hp, W0, a.n_examples, seed=11)
        dist.barrier()
        if rank == 0:
            Wr, _ = A.replay(res.events, plan, CudaBackend(prob, a.batch // plan.k), hp, W0,
                             a.n_examples, seed=11)
            burn = min(3 * g + 5, len(res.events) // 3)
            wt = res.write_times[burn:]
            st = np.array([e.staleness for e in res.events[burn:]])
            v, c = np.unique(st, return_counts=True)
            rows.append({
                "N": N, "g": g, "k": plan.k, "group_batch": a.batch, "updates": a.updates,
                "measured_s_per_update": float(np.diff(wt).mean()),
                "he_predict_s_per_update": he_predict(plan, profile),
                "t_conv_k": t_conv(plan.k, profile),
                "images_per_s": a.batch / float(np.diff(wt).mean()),
                "staleness_mean": float(st.mean()), "staleness_hist": {int(x): int(y) for x, y in zip(v, c)},
                "replay_max_abs_diff": float((Wr - res.W).abs().max()),
                "replay_bit_exact": bool(torch.equal(Wr, res.W)),
            })
            print(json.dumps(rows[-1]), flush=True)
    if rank == 0:
        out = {"net": a.net, "profile": {"T_cc": profile.T_cc, "T_nc": profile.T_nc, "t_fc": profile.t_fc},
               "profile_source": "T_cc: CUDA events, one GPU, group batch; T_nc: one-way P2P of the "
                                 "model (NCCL); t_fc: server update + reply", "rows": rows}
        print(json.dumps(out["profile"]))
        if a.out:
            with open(a.out, "w") as f:
                json.dump(out, f, indent=1)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
