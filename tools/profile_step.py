"""One training step inside an NVTX range "step", for ncu launch lists:

    ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,\
        dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python tools/profile_step.py caffenet 256

Warm-up steps run outside the range (lazy setup, attribute calls); the
profiled step is eager (no CUDA graph) so every launch is its own record.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_04487_b200 as P  # noqa: E402
from paper_1606_04487_b200.problems import CNNProblem, DeviceBatch  # noqa: E402


def main():
    net = sys.argv[1] if len(sys.argv) > 1 else "caffenet"
    b = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    prec = sys.argv[3] if len(sys.argv) > 3 else "tf32"
    prob = CNNProblem(net, n_examples=max(2 * b, 512), seed=0, precision=prec)
    hp = P.Hyperparams(eta=0.01, mu=0.9, lam=5e-4, b=b)
    sess = prob.device_session(prob.initial_state(), hp, use_graph=False)
    gen = torch.Generator(device="cuda").manual_seed(0)
    idx = [torch.randint(0, prob._n, (b,), device="cuda", generator=gen) for _ in range(4)]
    for i in range(3):
        sess.step(DeviceBatch(idx[i]))
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("step")
    sess.step(DeviceBatch(idx[3]))
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print(f"{net} b={b} {prec}: loss {sess.last_loss():.4f}")


if __name__ == "__main__":
    main()
