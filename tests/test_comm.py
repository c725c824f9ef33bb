"""The communicator entry points of the C-ABI (include/omni.h "comm"):
NCCL resolves at run time, ids have the declared size, argument errors map to
ValueError before any device call.  CPU only."""

import pytest

from paper_1606_04487_b200 import comm


def test_nccl_resolves():
    v = comm.nccl_version()
    assert v >= 22700, v                      # 2.27 (system) or 2.28 (torch's)


def test_unique_id_size_and_freshness():
    a, b = comm.unique_id(), comm.unique_id()
    assert len(a) == comm.ID_BYTES == 128
    assert a != b


def test_argument_errors_are_valueerror():
    uid = comm.unique_id()
    with pytest.raises(ValueError, match="outside"):
        comm.Communicator.init_rank(2, uid, 5, 0)
    with pytest.raises(ValueError, match="unique id"):
        comm.Communicator.init_rank(2, uid[:10], 0, 0)
    with pytest.raises(ValueError, match="NULL"):
        comm._abi.call("omni_allreduce_sum_f32", None, None, 4, None)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
def test_owned_parts_tile_each_slice(n):
    for lo, hi in [(0, 34848), (34848, 34944), (7, 8), (5, 5), (0, 37_748_736), (101, 4197)]:
        parts = [comm.owned_part(lo, hi, n, r) for r in range(n)]
        covered = []
        for a, b in parts:
            assert lo <= a <= b <= hi
            covered.extend(range(a, b)) if hi - lo < 100_000 else None
        if hi - lo < 100_000:
            assert covered == list(range(lo, hi))          # disjoint, in rank order, complete
        assert sum(b - a for a, b in parts) == hi - lo
        for a, b in parts:
            assert b == a or (a - lo) % 4 == 0                 # whole float4s from lo
