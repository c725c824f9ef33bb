"""Throughput of the free-running compute groups with the co-located server
(colocated.py) on N GPUs: CaffeNet, b images per GPU per gradient.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/async_colocated_bench.py [g] [T] [b] [net]

Prints one JSON line from rank 0: seconds per master update, images/s
(every update consumes one group batch of k*b images), the staleness
statistics, and cluster.he_predict / he_predict_pipelined / fc_saturated of the
phase times measured on this box (the HE check).
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1606_04487_b200 import colocated as C  # noqa: E402
from paper_1606_04487_b200.cluster import (ExecutionPlan, PhaseProfile, fc_saturated,  # noqa: E402
                                            he_predict, he_predict_pipelined)
from paper_1606_04487_b200.groups import CudaBackend  # noqa: E402
from paper_1606_04487_b200.problems import CNNProblem  # noqa: E402
from paper_1606_04487_b200.sgd import Hyperparams  # noqa: E402


def event_s(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def phase_profile(backend, prob, W0, hp, b, dev, world):
    """The iteration-time model's three scalars measured on this box (cluster.py:16-99):
    T_cc per GPU batch = one GPU's gradient of b images (CUDA events; the group
    batch of k GPUs is k b, so T_cc / k is this); T_nc = one-way NVLink copy of
    the whole model to a peer GPU (the runtime's gradient push / snapshot pull);
    t_fc = the server's service per update: the model's momentum update plus the
    snapshot copy back (simulator.py:170-205)."""
    idx = np.arange(b) % 1024
    T = event_s(lambda: backend.grad(W0, idx))
    peer = torch.device("cuda", (dev.index + 1) % torch.cuda.device_count()) if world > 1 else dev
    buf = torch.empty_like(W0, device=peer)
    T_nc = event_s(lambda: buf.copy_(W0, non_blocking=True))
    V = torch.zeros_like(W0)
    Wt, G, snap = W0.clone(), 0.001 * torch.ones_like(W0), W0.clone()
    svc = event_s(lambda: (backend.sgd(Wt, V, G, snap, hp), snap.copy_(Wt)))
    return {"T_cc_per_gpu_batch": T, "T_nc": T_nc, "server_update": svc, "t_fc": svc + T_nc}


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    g = int(sys.argv[1]) if len(sys.argv) > 1 else world
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 60
    b = int(sys.argv[3]) if len(sys.argv) > 3 else 256
    net = sys.argv[4] if len(sys.argv) > 4 else "caffenet"
    plan = ExecutionPlan(world, g)
    prob = CNNProblem(net, n_examples=1024, seed=rank, labels="uniform", precision="tf32", device=dev)
    hp = Hyperparams(eta=0.01, mu=0.9, lam=5e-4, b=b * plan.k)
    backend = CudaBackend(prob, b)
    gen = torch.Generator(device=dev).manual_seed(0)
    W0 = 0.01 * torch.randn(prob.dim, generator=gen, device=dev)
    C.run_colocated(plan, backend, hp, W0, 1024, 1, max(2 * g, 8))      # warm-up (lazy setup, graphs)
    torch.cuda.synchronize()
    res = C.run_colocated(plan, backend, hp, W0, 1024, 1, T)
    prof = phase_profile(backend, prob, W0, hp, b, dev, world) if rank == 0 else None
    if rank == 0:
        ev = res.events
        st = np.array([e.staleness for e in ev[g:]]) if len(ev) > g else np.array([0])
        wt = np.array([e.arrive_time for e in ev])
        per = float(np.diff(wt[g:]).mean()) if len(wt) > g + 1 else res.seconds / T
        print(json.dumps({"net": net, "N": world, "g": g, "k": plan.k, "per_gpu_batch": b,
                          "updates": T, "seconds": res.seconds, "s_per_update": per,
                          "images_per_s": hp.b / per, "staleness_mean": float(st.mean()),
                          "staleness_hist": {int(v): int((st == v).sum()) for v in np.unique(st)},
                          "phase_profile": prof,
                          "he_predict_s_per_update": he_predict(plan, PhaseProfile(
                              T_cc=prof["T_cc_per_gpu_batch"] * plan.k, T_nc=prof["T_nc"], t_fc=prof["t_fc"])),
                          "he_predict_pipelined_s_per_update": he_predict_pipelined(plan, PhaseProfile(
                              T_cc=prof["T_cc_per_gpu_batch"] * plan.k, T_nc=prof["T_nc"], t_fc=prof["t_fc"])),
                          "fc_saturated": fc_saturated(plan, PhaseProfile(
                              T_cc=prof["T_cc_per_gpu_batch"] * plan.k, T_nc=prof["T_nc"], t_fc=prof["t_fc"])),
                          "transport": "server co-located on rank 0; gradients/snapshots by copy-engine DMA "
                                       "over NVLink (IPC), shared-memory mailbox, group allreduce/broadcast "
                                       "on the C-ABI NCCL communicators"}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
