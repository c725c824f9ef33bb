"""The fused peer-memory reduce + momentum update (csrc/peer.cu) alone, on a
CaffeNet-sized parameter vector (62.4 M floats), against NCCL allreduce
followed by the separate update kernel.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/p2p_probe.py

Per rank and element of its part: N gradient loads (N-1 remote), V, W
loads, V, W stores, N-1 remote W stores.  Reported: time per full-vector
update (max over ranks, CUDA events), NVLink bytes per rank
(2 (N-1)/N * 4 * dim, read + written), and exactness of W across ranks."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1606_04487_b200 import comm  # noqa: E402
from paper_1606_04487_b200 import kernels as K  # noqa: E402

DIM = 62_378_344


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    z.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(z) / reps], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t)


def main():
    os.environ.setdefault("NCCL_NVLS_ENABLE", "0")
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    gen = torch.Generator(device=dev).manual_seed(rank)
    G = torch.randn(DIM, generator=gen, device=dev)
    W = torch.full((DIM,), 0.5, device=dev)
    V = torch.zeros(DIM, device=dev)
    peer = comm.PeerUpdate(G, W, 4, dist.group.WORLD, mode=os.environ.get("OMNI_P2P_MODE", "dma"))

    def fused():
        peer.begin_step()
        peer.layer(0, DIM, V, W, 1e-3 / world, 0.9, 5e-4 * world)
        peer.finish()

    ms_fused = timed(fused)
    # kernel alone (signals already satisfied): same launch without the waits
    a, b = peer.part(0, DIM)
    s = torch.cuda.current_stream()
    import ctypes
    from paper_1606_04487_b200 import _abi

    def kernel_only():
        _abi.call("omni_p2p_reduce_sgd_f32", peer.g_ptrs, peer.w_ptrs, world, rank, a, b,
                  ctypes.c_void_p(V.data_ptr()), ctypes.c_void_p(W.data_ptr()),
                  1e-3 / world, 0.9, 5e-4 * world, ctypes.c_void_p(s.cuda_stream))

    ms_kernel = timed(kernel_only) if peer.mode == "pull" else float("nan")
    Gc = G.clone()

    def nccl():
        Gc.copy_(G)
        dist.all_reduce(Gc)
        K.sgd_momentum(W, V, Gc, W, 1e-3 / world, 0.9, 5e-4 * world)

    ms_nccl = timed(nccl)
    ms_copy = timed(lambda: Gc.copy_(G))
    fused()
    torch.cuda.synchronize()
    sums = [None] * world
    dist.all_gather_object(sums, float(W.double().sum()))
    nvlink = 2 * (world - 1) / world * 4 * DIM
    out = {"world": world, "dim": DIM, "fused_ms": ms_fused, "fused_kernel_ms": ms_kernel,
           "nccl_allreduce_plus_update_ms": ms_nccl - ms_copy, "nvlink_bytes_per_rank": nvlink,
           "fused_kernel_nvlink_GBps": nvlink / (ms_kernel * 1e6),
           "W_identical_on_all_ranks": len(set(sums)) == 1, "mode": peer.mode}
    if rank == 0:
        print(json.dumps(out), flush=True)
    peer.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
