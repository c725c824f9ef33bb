"""Data-parallel DeviceSession (N ranks, per-layer async allreduce + layer-wise
update inside the backward) == the synchronous update on the mean gradient.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/dp_check.py

Every rank steps on its own batch; afterwards rank 0 recomputes each rank's
gradient with the same engine (same kernels, same batches) step by step and
applies V = mu V - eta (mean_r G_r + lam W); W += V in float64.  Prints the
normwise difference of the final W (fp32 session vs fp64 replay of the same
fp32 gradients).
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
        W = np.asarray(state.W, dtype=np.float64).copy()
        V = np.zeros_like(W)
        eng = prob.engine(b)
        for t in range(steps):
            Wd = torch.from_numpy(W.astype(np.float32)).to(dev)
            G = np.zeros_like(W)
            for r in range(world):
                eng.gather_batch(prob.data, prob.data_labels, torch.from_numpy(idx[t][r]).to(dev))
                _, g = eng.loss_and_grad(Wd, b)
                G += g.double().cpu().numpy() / world
            V = hp.mu * V - hp.eta * (G + hp.lam * W)
            W = W + V
        rel = float(np.linalg.norm(W_dp - W) / np.linalg.norm(W))
        relv = float(np.linalg.norm(st.V - V) / np.linalg.norm(V))
        print(f"{net}: N={world} data-parallel{' merged-FC' if merged else ' p2p' if p2p else ''} session vs replay: "
              f"normwise {rel:.3e}, V {relv:.3e} (last loss {loss:.4f})")
        worst = []
        for op in eng.ops:
            if op.kind in ("conv", "fc"):
                hi = op.boff + op.layer.d_out if op.boff >= 0 else op.woff + op.wsz
                for nm, lo, h in (("w", op.woff, op.woff + op.wsz), ("b", op.boff, hi)):
                    if h > lo >= 0:
                        e = float(np.linalg.norm(st.V[lo:h] - V[lo:h]) / max(np.linalg.norm(V[lo:h]), 1e-30))
                        worst.append((e, f"{op.kind}@{op.woff}.{nm}[{h - lo}]"))
        print("worst V slices:", sorted(worst, reverse=True)[:4])
        assert rel < 1e-5 and relv < 1e-2, (rel, relv)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
