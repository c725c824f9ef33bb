"""Is the e2e gap interference from the concurrent host->device copy?  Times the
device-batch training loop alone and with a background 158 MB pinned H2D copy
per step (into a dummy buffer, on its own stream).

    python tools/e2e_probe.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1606_04487_b200.problems import CNNProblem, DeviceBatch  # noqa: E402
from paper_1606_04487_b200.sgd import Hyperparams, SGDState  # noqa: E402


def main():
    b, steps = 256, 30
    prob = CNNProblem("caffenet", n_examples=1024, seed=0, labels="uniform", precision="tf32")
    sess = prob.device_session(SGDState.fresh(np.zeros(1)), Hyperparams(eta=0.01, mu=0.9, lam=5e-4, b=b))
    sess.W = 0.01 * torch.randn(prob.dim, device="cuda")
    sess.V = torch.zeros_like(sess.W)
    idx = torch.randint(0, 1024, (steps + 5, b), device="cuda")
    host = torch.randn(b, 227, 227, 3).pin_memory()
    dummy = torch.empty(host.shape, device="cuda")
    cs = torch.cuda.Stream()
    for i in range(5):
        sess.step(DeviceBatch(idx[i]))
    for copy in (False, True, False, True):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(steps):
            if copy:
                with torch.cuda.stream(cs):
                    dummy.copy_(host, non_blocking=True)
            sess.step(DeviceBatch(idx[5 + i % steps]))
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        print(f"background H2D copy {copy}: {ms:.3f} ms/step, {b / ms * 1e3:.0f} img/s")


if __name__ == "__main__":
    main()
