"""Data-parallel DeviceSession (N ranks, per-layer async allreduce + layer-wise
update inside the backward; or the peer-memory fused reduce + update; or
merged FC) == the synchronous update on the mean gradient, replayed by the
float64 CPU ORACLE.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/mp_dp_check.py [net] [p2p|merged]

Every rank steps on its own batch; afterwards rank 0 replays the run on the
host: each rank's batch gradient from oracle/refcnn.grad (float64, the
reference's algorithm, problems.py:239-269) at the replayed W, the mean over
ranks, and V = mu V - eta (mean_r G_r + lam W); W += V (sgd.py:92-101).  The
fp32 session must match that replay (final W normwise <= 1e-4, the learned
update W_T - W_0 and V_T <= 1e-3 in 3xTF32).
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import refcnn as R  # noqa: E402
from paper_1606_04487_b200.problems import CNNProblem, DeviceBatch  # noqa: E402
from paper_1606_04487_b200.sgd import Hyperparams, SGDState  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    net = sys.argv[1] if len(sys.argv) > 1 else "cifar10_quick"
    merged = len(sys.argv) > 2 and sys.argv[2] == "merged"
    p2p = len(sys.argv) > 2 and sys.argv[2] == "p2p"
    b, steps = 32, 4
    prob = CNNProblem(net, n_examples=256, seed=3, precision="3xtf32", device=dev)
    hp = Hyperparams(eta=0.01, mu=0.9, lam=5e-4, b=b)
    state = prob.initial_state()
    rng = np.random.default_rng(11)
    idx = [[rng.integers(0, 256, size=b) for _ in range(world)] for _ in range(steps)]
    sess = prob.device_session(state, hp, process_group=dist.group.WORLD, merged_fc=merged,
                                p2p=p2p)
    for t in range(steps):
        sess.step(DeviceBatch(torch.from_numpy(idx[t][rank]).to(dev)))
    loss = sess.last_loss()            # (merged FC: a collective)
    sess.sync_fc()
    torch.cuda.synchronize()
    W_dp = sess.W.double().cpu().numpy()
    st = sess.state()                  # (p2p: gathers V, a collective)
    Ws = [None] * world
    dist.all_gather_object(Ws, float(np.abs(W_dp).sum()))
    if p2p:                            # one owner computes each element: bit-identical W
        assert len(set(Ws)) == 1, Ws
    if rank == 0:
        W0 = np.asarray(state.W, dtype=np.float32).astype(np.float64)
        W, V = W0.copy(), np.zeros_like(W0)
        images = prob.images.astype(np.float32).astype(np.float64)
        L = prob.net.to_dicts()
        with R.gemm_impl("blas"):
            for t in range(steps):
                G = np.zeros_like(W)
                for r in range(world):
                    ix = idx[t][r]
                    G += R.grad(L, prob.net.in_channels, prob.net.in_size, W, images[ix], prob.labels[ix]) / world
                W, V = R.sgd_step(W, V, G, W, hp.eta, hp.mu, hp.lam)
        rel = float(np.linalg.norm(W_dp - W) / np.linalg.norm(W))
        reld = float(np.linalg.norm((W_dp - W0) - (W - W0)) / np.linalg.norm(W - W0))
        relv = float(np.linalg.norm(st.V - V) / np.linalg.norm(V))
        print(f"{net}: N={world} data-parallel{' merged-FC' if merged else ' p2p' if p2p else ''} session vs "
              f"oracle replay: W normwise {rel:.3e}, W_T - W_0 {reld:.3e}, V {relv:.3e} (last loss {loss:.4f})")
        assert rel < 1e-4 and reld < 1e-3 and relv < 1e-3, (rel, reld, relv)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
