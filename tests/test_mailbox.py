"""The co-located server's shared-memory mailbox (csrc/mailbox.cu) across
processes: tickets come out in the order they were taken (FIFO by arrival,
the serial server of simulator.py:3-7), every group's posts are consumed
exactly once, snapshot sequences and the stop value reach the waiting
leaders, and waits time out instead of hanging."""

import ctypes
import multiprocessing as mp
import os
import uuid

import pytest

from paper_1606_04487_b200 import _abi


def _open(name):
    box = ctypes.c_void_p()
    _abi.call("omni_mailbox_open", name.encode(), ctypes.byref(box), 10_000)
    return box


def _leader(name, g, n, q):
    box = _open(name)
    last, tickets = 0, []
    for _ in range(n):
        t = ctypes.c_longlong()
        _abi.call("omni_mailbox_post", box, g, ctypes.byref(t))
        tickets.append(t.value)
        s = ctypes.c_longlong()
        _abi.call("omni_mailbox_snap_wait", box, g, last, ctypes.byref(s), 10_000)
        last = s.value
        if last < 0:
            break
    q.put((g, tickets, last))
    _abi.call("omni_mailbox_close", box, None)


def test_mailbox_fifo_exactly_once_and_stop():
    name = f"/omni_test_{uuid.uuid4().hex[:12]}"
    box = ctypes.c_void_p()
    G, T = 3, 60
    _abi.call("omni_mailbox_create", name.encode(), G, ctypes.byref(box))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_leader, args=(name, g, 1000, q)) for g in range(G)]
    for p in ps:
        p.start()
    seq = [0] * G
    order = []
    for t in range(T):
        g = ctypes.c_int()
        _abi.call("omni_mailbox_next", box, ctypes.byref(g), 10_000)
        order.append(g.value)
        seq[g.value] += 1
        _abi.call("omni_mailbox_snap_post", box, g.value, seq[g.value])
    for _ in range(G):                       # drain: each group's pending post, then stop
        g = ctypes.c_int()
        _abi.call("omni_mailbox_next", box, ctypes.byref(g), 10_000)
        order.append(g.value)
        _abi.call("omni_mailbox_snap_post", box, g.value, -1)
    res = {}
    for _ in range(G):
        g, tickets, last = q.get(timeout=30)
        res[g] = (tickets, last)
    for p in ps:
        p.join(30)
        assert p.exitcode == 0
    _abi.call("omni_mailbox_close", box, name.encode())
    # every post consumed exactly once, in ticket order
    all_tickets = sorted((t, g) for g, (ts, _) in res.items() for t in ts)
    assert [t for t, _ in all_tickets] == list(range(T + G))
    assert [g for _, g in all_tickets] == order
    assert all(last == -1 for _, last in res.values())
    assert sum(len(ts) for ts, _ in res.values()) == T + G


def test_mailbox_waits_time_out():
    name = f"/omni_test_{uuid.uuid4().hex[:12]}"
    box = ctypes.c_void_p()
    _abi.call("omni_mailbox_create", name.encode(), 2, ctypes.byref(box))
    g = ctypes.c_int()
    with pytest.raises(RuntimeError, match="no gradient"):
        _abi.call("omni_mailbox_next", box, ctypes.byref(g), 50)
    s = ctypes.c_longlong()
    with pytest.raises(RuntimeError, match="no snapshot"):
        _abi.call("omni_mailbox_snap_wait", box, 1, 0, ctypes.byref(s), 50)
    with pytest.raises(ValueError):
        _abi.call("omni_mailbox_post", box, 5, None)
    _abi.call("omni_mailbox_close", box, name.encode())
    other = ctypes.c_void_p()
    with pytest.raises(RuntimeError, match="not created"):
        _abi.call("omni_mailbox_open", f"/omni_missing_{os.getpid()}".encode(), ctypes.byref(other), 50)
