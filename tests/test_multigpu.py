"""Multi-GPU parity checks (NCCL, one process per GPU), run through torchrun
when the box has >= 2 GPUs (skipped on single-GPU boxes):

* data-parallel DeviceSession (per-layer async allreduce, layer-wise update;
  peer-memory fused reduce + update; merged FC) == the float64 ORACLE replay
  (refcnn.grad of every rank's batch, mean, sgd.py:92-101 update);
* the round-synchronous compute-group runtime == the oracle's deterministic
  simulate (event log and weights)."""

import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def torchrun(n, script, *args, env=None):
    # the checkers that import the oracle live under tests/ (mp_*.py); probes under tools/
    where = "tests" if script.startswith("mp_") else "tools"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}",
           os.path.join(ROOT, where, script), *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env=None if env is None else {**os.environ, **env})
    if r.returncode != 0:
        # the failing rank's traceback sits before torchrun's own summary
        tb = [ln for ln in r.stderr.splitlines() if not ln.startswith(("E1", "W1", "I1"))]
        raise AssertionError(r.stdout[-3000:] + "\n".join(tb)[-8000:])
    return r.stdout


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("mode", ["", "merged", "p2p"])
def test_data_parallel_session_equals_replay(mode):
    out = torchrun(2, "mp_dp_check.py", "cifar10_quick", *([mode] if mode else []))
    assert "normwise" in out


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("mode", ["", "--p2p", "--overlap", "--replicated"])
def test_group_runtime_equals_oracle_schedule(mode):
    out = torchrun(2, "mp_groups_check.py", *([mode] if mode else []))
    assert '"pass": true' in out


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_c_abi_communicators_one_process_per_gpu():
    out = torchrun(2, "comm_check.py")
    assert '"pass": true' in out


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("transport", ["dma", "pull"])
def test_peer_memory_update_both_transports(transport):
    """mp_dp_check asserts W bit-identical on every rank and equal to the
    float64 oracle replay."""
    out = torchrun(2, "mp_dp_check.py", "lenet", "p2p", env={"OMNI_P2P_MODE": transport})
    assert "p2p session vs oracle replay" in out


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_peer_update_probe_exact():
    out = torchrun(2, "p2p_probe.py")
    assert '"W_identical_on_all_ranks": true' in out


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("g", [1, 2])
def test_colocated_async_groups_two_gpus(g):
    """Free-running groups, server co-located on rank 0 (no extra GPU):
    valid schedule, bit-exact replay, float64 oracle replay <= 1e-4."""
    out = torchrun(2, "mp_async_check.py", "cifar10_quick", str(g), "16")
    assert '"pass": true' in out


@pytest.mark.skipif(NGPU < 4, reason="needs >= 4 GPUs")
@pytest.mark.parametrize("g", [2, 4])
def test_colocated_async_groups_four_gpus(g):
    out = torchrun(4, "mp_async_check.py", "cifar10_quick", str(g), "16")
    assert '"pass": true' in out
