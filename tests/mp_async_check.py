"""Free-running compute groups with the co-located server (colocated.py) on
N GPUs, checked on rank 0:

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/mp_async_check.py [net] [g] [T]

* the update log is a valid asynchronous schedule (FIFO write steps 1..T,
  each group reads the model right after its own previous write, staleness =
  write - 1 - read);
* replaying the log with the same kernels reproduces the server's final
  model (bit for bit for k <= 2);
* replaying the log in the float64 ORACLE (refcnn.grad at each group's stale
  snapshot, sgd_step with that snapshot as w_read: simulator.py:170-205,
  sgd.py:104-112) lands within 1e-4 of it -- the asynchronous update
  semantics are the reference's;
* the staleness statistics (mean ~ g - 1 for equal groups).
Prints one JSON line (seconds per update, images/s, staleness).
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import refcnn as R  # noqa: E402
from paper_1606_04487_b200 import async_groups as A, colocated as C  # noqa: E402
from paper_1606_04487_b200.cluster import ExecutionPlan  # noqa: E402
from paper_1606_04487_b200.groups import CudaBackend  # noqa: E402
from paper_1606_04487_b200.problems import CNNProblem  # noqa: E402
from paper_1606_04487_b200.sgd import Hyperparams, batch_stream  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    net = sys.argv[1] if len(sys.argv) > 1 else "cifar10_quick"
    g = int(sys.argv[2]) if len(sys.argv) > 2 else world
    T = int(sys.argv[3]) if len(sys.argv) > 3 else 16
    per, n_ex, seed = 32, 256, 11
    prob = CNNProblem(net, n_examples=n_ex, seed=3, precision="3xtf32", device=dev)
    plan = ExecutionPlan(world, g)
    hp = Hyperparams(eta=0.01, mu=0.5, lam=5e-4, b=per * plan.k)
    backend = CudaBackend(prob, per)
    W0 = torch.from_numpy(prob.initial_weights().astype(np.float32)).to(dev)
    res = C.run_colocated(plan, backend, hp, W0, n_ex, seed, T)
    if rank == 0:
        ev = np.array([[e.group_id, e.read_step, e.write_step, e.staleness, e.batch_index] for e in res.events])
        assert ev.shape[0] == T and np.array_equal(ev[:, 2], np.arange(1, T + 1))
        assert np.array_equal(ev[:, 3], ev[:, 2] - 1 - ev[:, 1]) and (ev[:, 3] >= 0).all()
        for i in range(g):
            mine = ev[ev[:, 0] == i]
            assert len(mine) > 0 and mine[0, 1] == 0
            assert np.array_equal(mine[:, 4], np.arange(len(mine)))
            assert np.array_equal(mine[1:, 1], mine[:-1, 2])
        Wr, _ = A.replay(res.events, plan, backend, hp, W0, n_ex, seed)
        exact = bool(torch.equal(Wr, res.W))
        if plan.k <= 2:
            assert exact, float((Wr - res.W).abs().max())
        # the same log in the float64 oracle
        images = prob.images.astype(np.float32).astype(np.float64)
        L = prob.net.to_dicts()
        Wo = W0.double().cpu().numpy()
        Vo = np.zeros_like(Wo)
        snaps = [Wo.copy() for _ in range(g)]
        rngs = [batch_stream(seed, i) for i in range(g)]
        with R.gemm_impl("blas"):
            for e in res.events:
                idx = rngs[e.group_id].integers(0, n_ex, size=hp.b)
                G = sum(R.grad(L, prob.net.in_channels, prob.net.in_size, snaps[e.group_id],
                               images[idx[m * per:(m + 1) * per]], prob.labels[idx[m * per:(m + 1) * per]])
                        for m in range(plan.k))
                Wo, Vo = R.sgd_step(Wo, Vo, G, snaps[e.group_id], hp.eta / plan.k, hp.mu, hp.lam * plan.k)
                snaps[e.group_id] = Wo.copy()
        W = res.W.double().cpu().numpy()
        rel = float(np.linalg.norm(W - Wo) / np.linalg.norm(Wo))
        reld = float(np.linalg.norm((W - Wo)) / max(np.linalg.norm(Wo - W0.double().cpu().numpy()), 1e-300))
        assert rel < 1e-4, rel
        st = ev[g:, 3] if T > g else ev[:, 3]
        print(json.dumps({"net": net, "N": world, "g": g, "k": plan.k, "updates": T,
                          "seconds": res.seconds, "s_per_update": res.seconds / T,
                          "images_per_s": T * hp.b / res.seconds,
                          "staleness_mean_after_warmup": float(np.mean(st)),
                          "replay_bit_exact": exact, "oracle_replay_rel_W": rel,
                          "oracle_replay_rel_update": reld, "pass": True}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
