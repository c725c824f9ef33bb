"""One process per GPU through the C-ABI communicators (no torch NCCL on the
data path): rank 0 makes the NCCL id, the torch store ships it, every rank
calls omni_comm_init_rank; then a CaffeNet-sized gradient allreduce (exact on
integer data, timed), a split into the compute groups of ExecutionPlan(N, g),
a server <-> leader snapshot exchange, an all-gather and a personalised
all-to-all (the sharded group runtime's exchanges).

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/comm_check.py
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1606_04487_b200 import comm  # noqa: E402
from paper_1606_04487_b200.cluster import ExecutionPlan  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")                  # id exchange only
    obj = [comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    c = comm.Communicator.init_rank(world, obj[0], rank, rank)
    out = {"world": world, "nccl": comm.nccl_version()}

    n = 62_378_344                                    # CaffeNet parameters
    g = torch.full((n,), float(rank + 1), device="cuda")
    c.allreduce_sum(g)
    torch.cuda.synchronize()
    out["allreduce_exact"] = bool(torch.all(g == world * (world + 1) / 2).item())
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        c.allreduce_sum(g)
    a.record()
    reps = 10
    for _ in range(reps):
        c.allreduce_sum(g)
    z.record()
    torch.cuda.synchronize()
    ms = torch.tensor([a.elapsed_time(z) / reps])
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    out["allreduce_ms"] = float(ms)
    out["busbw_GBps"] = 4 * n * 2 * (world - 1) / world / (float(ms) * 1e6)

    # server (rank 0) <-> every other rank: snapshot out, gradient back
    snap = torch.full((1 << 20,), 7.0, device="cuda") if rank == 0 else torch.zeros(1 << 20, device="cuda")
    if rank == 0:
        grads = [torch.zeros(1 << 20, device="cuda") for _ in range(world - 1)]
        with comm.group():
            for p in range(1, world):
                c.send(snap, p)
                c.recv(grads[p - 1], p)
        torch.cuda.synchronize()
        out["p2p_exact"] = all(bool(torch.all(gr == 7.0 + p).item()) for p, gr in enumerate(grads, 1))
    elif world > 1:                               # (one fused send+recv pair, like the server)
        grad = torch.full((1 << 20,), 7.0 + rank, device="cuda")
        with comm.group():
            c.recv(snap, 0)
            c.send(grad, 0)
        torch.cuda.synchronize()
        assert bool(torch.all(snap == 7.0).item())
    # all-gather and the personalised all-to-all (parts from scattered addresses)
    m = 1000
    ag = torch.empty(world * m, device="cuda")
    c.allgather(torch.full((m,), float(rank), device="cuda"), ag)
    pool = torch.arange(world * 2 * m, dtype=torch.float32, device="cuda") + 1e4 * rank
    parts = [pool[(2 * d + 1) * m:(2 * d + 2) * m] for d in range(world)]   # non-adjacent parts
    recv = torch.empty(world * m, device="cuda")
    c.all_to_all(parts, recv)
    torch.cuda.synchronize()
    want_ag = torch.arange(world, device="cuda").float().repeat_interleave(m)
    out["allgather_exact"] = bool(torch.equal(ag, want_ag))
    want = torch.cat([torch.arange((2 * rank + 1) * m, (2 * rank + 2) * m, device="cuda").float() + 1e4 * src
                      for src in range(world)])
    out["all_to_all_exact"] = bool(torch.equal(recv, want))
    for groups in [d for d in (1, 2, 4, 8) if world % d == 0]:
        k = ExecutionPlan(world, groups).k
        s = c.split(rank // k, rank % k)
        x = torch.full((1 << 20,), float(rank), device="cuda")
        s.allreduce_sum(x)
        torch.cuda.synchronize()
        grp = rank // k
        ok = bool(torch.all(x == float(sum(range(grp * k, grp * k + k)))).item())
        out[f"split_g{groups}_exact"] = ok and s.size_rank() == (k, rank % k)
        s.destroy()

    c.destroy()
    if rank == 0:
        out["pass"] = all(v for kk, v in out.items() if kk.endswith("exact"))
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
