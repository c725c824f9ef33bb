"""Communicators through the C-ABI on real GPUs: one process driving every
visible device (omni_comm_init_all), group split (one communicator per
compute group of an ExecutionPlan), in-place allreduce and point-to-point.
Results are exact: every value is a small integer in float32."""

import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_1606_04487_b200 import comm  # noqa: E402
from paper_1606_04487_b200.cluster import ExecutionPlan  # noqa: E402


def _comms():
    n = torch.cuda.device_count()
    return n, comm.Communicator.init_all(list(range(n)))


def test_init_all_allreduce_exact():
    n, cs = _comms()
    assert [c.size_rank() for c in cs] == [(n, i) for i in range(n)]
    bufs = [torch.arange(1000, dtype=torch.float32, device=f"cuda:{i}") * (i + 1) for i in range(n)]
    with comm.group():
        for c, b in zip(cs, bufs):
            with torch.cuda.device(c.device):
                c.allreduce_sum(b)
    want = torch.arange(1000, dtype=torch.float32) * (n * (n + 1) // 2)
    for b in bufs:
        torch.cuda.synchronize(b.device)
        assert torch.equal(b.cpu(), want)
    z = torch.empty(0, device="cuda:0")
    cs[0].allreduce_sum(z)                   # empty: no-op
    for c in cs:
        c.destroy()


def test_split_into_compute_groups():
    n, cs = _comms()
    for g in [d for d in (1, 2, 4, 8) if n % d == 0]:
        plan = ExecutionPlan(n, g)
        k = plan.k
        with comm.group():
            subs = [c.split(i // k, i % k) for i, c in enumerate(cs)]
        for i, s in enumerate(subs):
            assert s.size_rank() == (k, i % k)
        bufs = [torch.full((257,), float(i), device=f"cuda:{i}") for i in range(n)]
        with comm.group():
            for s, b in zip(subs, bufs):
                with torch.cuda.device(s.device):
                    s.allreduce_sum(b)
        for i, b in enumerate(bufs):
            grp = i // k
            want = float(sum(range(grp * k, grp * k + k)))
            assert torch.equal(b.cpu(), torch.full((257,), want))
        for s in subs:
            s.destroy()
    for c in cs:
        c.destroy()


def test_send_recv_ring():
    n, cs = _comms()
    src = [torch.full((4096,), float(i + 1), device=f"cuda:{i}") for i in range(n)]
    dst = [torch.zeros(4096, device=f"cuda:{i}") for i in range(n)]
    with comm.group():
        for i, c in enumerate(cs):
            with torch.cuda.device(c.device):
                c.send(src[i], (i + 1) % n)
                c.recv(dst[i], (i - 1) % n)
    for i in range(n):
        torch.cuda.synchronize(i)
        assert torch.equal(dst[i].cpu(), torch.full((4096,), float((i - 1) % n + 1)))
    for c in cs:
        c.destroy()
