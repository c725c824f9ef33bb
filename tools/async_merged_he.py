"""Merged-FC free-running asynchronous groups on B200s (the paper's physical
mapping) + HE-model validation.  Rank 0 is the server and
owns the FC layers (FC staleness 0); ranks 1..g are single-GPU conv groups.

    torchrun --nproc-per-node P --master-addr 127.0.0.1 tools/async_merged_he.py \
        --updates 80 --out gpurun_out/async_merged.json

PhaseProfile measured on this box, in the reference's terms (cluster.py):
T_cc = one GPU's conv forward + backward for the group batch, T_nc = one-way
transfer of the conv model, t_fc = the server's FC forward + backward +
update for one group batch plus the activation and d(pool5) transfers.
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
from paper_1606_04487_b200 import kernels as K  # noqa: E402
from paper_1606_04487_b200 import nets  # noqa: E402
from paper_1606_04487_b200.cluster import ExecutionPlan, PhaseProfile, fc_saturated, he_predict  # noqa: E402
from paper_1606_04487_b200.engine import GpuNet  # noqa: E402
from paper_1606_04487_b200.problems import CNNProblem  # noqa: E402
from paper_1606_04487_b200.sgd import Hyperparams  # noqa: E402


def ev_ms(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    z.record()
    torch.cuda.synchronize()
    return a.elapsed_time(z) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="caffenet")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--updates", type=int, default=80)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    os.environ.setdefault("NCCL_NVLS_ENABLE", "0")
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    N = world - 1
    prob = CNNProblem(a.net, n_examples=1024, seed=5, labels="uniform", precision="tf32", device=dev)
    gen = torch.Generator(device=dev).manual_seed(7)
    W0 = 0.01 * torch.randn(prob.dim, generator=gen, device=dev)
    b = a.batch
    hp = Hyperparams(eta=0.01, mu=0.9, lam=5e-4, b=b)
    head_spec, fc_off = nets.fc_head(prob.net)
    eng = prob.engine(b)
    f = eng.first_fc
    act_shape = tuple(eng.ops[f].inp.value[:b].shape)
    head = GpuNet(head_spec, b, dev, "tf32", input_grad=True, input_cs=eng.ops[f].inp.cs) if rank == 0 else None

    # ---- PhaseProfile
    prof = {}
    if rank == 1:
        idx = torch.arange(b, device=dev) % 1024

        def conv_pass():
            eng.gather_batch(prob.data, prob.data_labels, idx)
            eng.forward(W0, b, stop=f)
            eng.backward(b, start=f)
        prof["T_cc"] = ev_ms(conv_pass) / 1e3
    dist.barrier()
    buf = torch.empty(fc_off, device=dev)
    abuf = torch.empty(act_shape, device=dev)
    if rank in (0, 1):
        times = {"model": [], "act": []}
        for rep in range(4):
            for key, x in (("model", W0[:fc_off].contiguous() if rank == 0 else buf),
                           ("act", abuf)):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                if rank == 0:
                    dist.send(x, dst=1)
                    dist.recv(x, src=1)
                else:
                    dist.recv(x, src=0)
                    dist.send(x, dst=0)
                torch.cuda.synchronize()
                if rep:
                    times[key].append((time.perf_counter() - t0) / 2)
        prof["T_nc"] = float(np.median(times["model"]))
        prof["act_xfer"] = float(np.median(times["act"]))
    if rank == 0:
        V = torch.zeros(prob.dim - fc_off, device=dev)
        Wfc = W0[fc_off:].clone()

        def fc_pass():
            head.forward(Wfc, b)
            head.backward(b)
            K.sgd_momentum(Wfc, V, head.grad, Wfc, hp.eta, hp.mu, hp.lam)
        prof["t_fc_compute"] = ev_ms(fc_pass) / 1e3
        prof["t_fc"] = prof["t_fc_compute"] + 2 * prof["act_xfer"]   # activations in, d(pool5) out
    dist.barrier()
    allp = [None] * world
    dist.all_gather_object(allp, prof)
    p0, p1 = allp[0], allp[1]
    profile = PhaseProfile(T_cc=p1["T_cc"], T_nc=p0["T_nc"], t_fc=p0["t_fc"])

    rows = []
    g = N                                           # one launch = g single-GPU groups (ranks 1..g)
    plan = ExecutionPlan(g, g)
    dist.barrier()
    if rank == 0:
        evs, W, Vm, secs = A.run_server_merged(plan, head, hp, W0, fc_off, act_shape, a.updates)
        Wr, _ = A.replay_merged(evs, plan, eng, head, prob, hp, W0, fc_off, seed=11)
        conv = [e for e in evs if e.kind == "conv"]
        burn = min(3 * g + 5, len(conv) // 3)
        wt = np.array([e.arrive_time for e in conv[burn:]])
        st = np.array([e.write_step - 1 - e.read_step for e in conv[burn:]])
        v, c = np.unique(st, return_counts=True)
        rows.append({
            "g": g, "group_batch": b, "updates": a.updates,
            "measured_s_per_update": float(np.diff(wt).mean()),
            "he_predict_s_per_update": he_predict(plan, profile),
            "fc_saturated_predicted": fc_saturated(plan, profile),
            "images_per_s": b / float(np.diff(wt).mean()),
            "conv_staleness_mean": float(st.mean()),
            "conv_staleness_hist": {int(x): int(y) for x, y in zip(v, c)},
            "fc_updates": sum(1 for e in evs if e.kind == "fc"),
            "replay_bit_exact": bool(torch.equal(Wr, W)),
            "replay_max_abs_diff": float((Wr - W).abs().max()),
        })
        print(json.dumps(rows[-1]), flush=True)
    else:
        A.run_worker_merged(plan, eng, prob, hp, W0, fc_off, seed=11)
    if rank == 0:
        out = {"net": a.net, "mapping": "merged FC on the server (rank 0), single-GPU conv groups",
               "profile": {"T_cc": profile.T_cc, "T_nc": profile.T_nc, "t_fc": profile.t_fc,
                           "t_fc_compute": p0["t_fc_compute"], "act_xfer": p0["act_xfer"]},
               "rows": rows}
        print(json.dumps(out["profile"]))
        if a.out:
            with open(a.out, "w") as fo:
                json.dump(out, fo, indent=1)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
