"""The reference SPEC's examples and invariants for the operator API
(SPEC.md module `conv`: conv_direct, lower, gemm, lift, conv_lowered,
blowup_ratio), run through this package's drop-in API on the GPU.

Tolerances: lowering / lift / blowup are exact (bit-identical float64 copies);
products run in 3xTF32 (fp32 accumulation), so where the SPEC states 1e-10
for the float64 reference, the bound here is 2e-6 normwise -- the same class
as test_parity_gpu.py -- and exact algebraic identities (identity kernel, zero
kernel) are checked at that bound or exactly where no rounding can occur."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1606_04487_b200 as P  # noqa: E402
from oracle import refcnn as R  # noqa: E402

TOL = 2e-6


def nrel(x, ref):
    return float(np.linalg.norm(np.asarray(x) - ref) / max(np.linalg.norm(ref), 1e-300))


def rand_case(rng, n, k, din, dout, b):
    D = rng.standard_normal((b, din, n, n)).astype(np.float32).astype(np.float64)
    K = rng.standard_normal((dout, din, k, k)).astype(np.float32).astype(np.float64)
    return D, K


def test_conv_direct_identity_zero_and_kat():
    rng = np.random.default_rng(0)
    D = rng.standard_normal((1, 1, 2, 2))
    spec = P.ConvSpec(n=2, k=1, d_in=1, d_out=1)
    assert nrel(P.conv_lowered(P.Tensor4(D), P.Tensor4(np.ones((1, 1, 1, 1))), spec).values, D) < TOL
    D3 = np.arange(1, 10, dtype=np.float64).reshape(1, 1, 3, 3)
    R2 = P.conv_lowered(P.Tensor4(D3), P.Tensor4(np.array([[1.0, 0.0], [0.0, 1.0]]).reshape(1, 1, 2, 2)),
                        P.ConvSpec(n=3, k=2, d_in=1, d_out=1)).values.reshape(2, 2)
    assert np.allclose(R2, [[6, 8], [12, 14]], atol=1e-5)
    Dz, _ = rand_case(rng, 7, 3, 2, 3, 2)
    Rz = P.conv_lowered(P.Tensor4(Dz), P.Tensor4(np.zeros((3, 2, 3, 3))), P.ConvSpec(n=7, k=3, d_in=2, d_out=3))
    assert np.array_equal(Rz.values, np.zeros_like(Rz.values))


@pytest.mark.parametrize("n,k,s,p,blow", [(5, 5, 1, 0, 1.0), (4, 3, 1, 0, 2.25), (6, 1, 1, 0, 1.0)])
def test_lower_shapes_and_blowup(n, k, s, p, blow):
    rng = np.random.default_rng(n * 10 + k)
    b, din = 3, 2
    D, _ = rand_case(rng, n, k, din, 1, b)
    spec = P.ConvSpec(n=n, k=k, d_in=din, d_out=1, stride=s, pad=p)
    L = P.lower(P.Tensor4(D), spec, b_p=b)
    m = (n + 2 * p - k) // s + 1
    assert L.matrix.shape == (b * m * m, k * k * din)
    assert P.blowup_ratio(spec) == blow
    assert L.matrix.size == blow * n * n * din * b                       # blowup accounting, exact
    assert np.array_equal(L.matrix, R.lower(D, k, s, p))                  # bit-exact
    if k == 1:                                                            # pure reshape of D
        assert np.array_equal(L.matrix, D.transpose(0, 2, 3, 1).reshape(b * n * n, din))


def test_gemm_examples():
    rng = np.random.default_rng(3)
    B = rng.standard_normal((2, 3))
    assert nrel(P.gemm(np.eye(2), B), B) < TOL
    assert np.allclose(P.gemm([[1.0, 2.0], [3.0, 4.0]], [[5.0], [6.0]]), [[17.0], [39.0]], atol=1e-4)
    A, Bm = rng.standard_normal((7, 5)), rng.standard_normal((5, 3))
    naive = np.array([[sum(A[i, r] * Bm[r, j] for r in range(5)) for j in range(3)] for i in range(7)])
    assert nrel(P.gemm(A, Bm), naive) < TOL
    with pytest.raises(ValueError):
        P.gemm(np.ones((2, 3)), np.ones((2, 3)))


def test_lift_examples():
    rng = np.random.default_rng(4)
    spec1 = P.ConvSpec(n=3, k=3, d_in=1, d_out=5)                        # m = 1
    Rh = rng.standard_normal((1, 5))
    assert np.array_equal(P.lift(Rh, spec1, 1).values.reshape(5), Rh.reshape(5))
    spec = P.ConvSpec(n=6, k=3, d_in=2, d_out=4, pad=1)
    assert np.array_equal(P.lift(np.zeros((2 * 36, 4)), spec, 2).values, np.zeros((2, 4, 6, 6)))
    D, K = rand_case(rng, 6, 3, 2, 4, 2)
    Rhat = P.gemm(P.lower(P.Tensor4(D), spec, b_p=2).matrix, P.lower_kernel(P.Tensor4(K), spec))
    assert nrel(P.lift(Rhat, spec, 2).values, R.conv_direct(D, K, 1, 1)) < TOL
    with pytest.raises(ValueError):
        P.lift(np.zeros((5, 4)), spec, 2)


def test_conv_lowered_partition_and_worker_invariance():
    rng = np.random.default_rng(5)
    D, K = rand_case(rng, 8, 3, 2, 4, 8)
    spec = P.ConvSpec(n=8, k=3, d_in=2, d_out=4)
    base = P.conv_lowered(P.Tensor4(D), P.Tensor4(K), spec, b_p=8, workers=1).values
    for b_p, workers in ((1, 1), (3, 1), (8, 4), (5, 2)):
        got = P.conv_lowered(P.Tensor4(D), P.Tensor4(K), spec, b_p=b_p, workers=workers).values
        assert np.array_equal(got, base), (b_p, workers)                  # bit-identical
    assert nrel(base, R.conv_direct(D, K)) < TOL
    # linearity and determinism
    assert nrel(P.conv_lowered(P.Tensor4(3.0 * D), P.Tensor4(K), spec, b_p=8).values, 3.0 * base) < TOL
    assert np.array_equal(P.conv_lowered(P.Tensor4(D), P.Tensor4(K), spec, b_p=8).values, base)


def test_oracle_equivalence_over_200_random_specs():
    """SPEC invariant: k in {1,2,3,5}, n <= 16, d_in, d_out <= 8, b <= 8, all b_p."""
    rng = np.random.default_rng(6)
    worst = 0.0
    done = 0
    while done < 200:
        k = int(rng.choice([1, 2, 3, 5]))
        s = int(rng.integers(1, 3))
        p = int(rng.integers(0, k))
        n = int(rng.integers(max(k, 2), 17))
        if (n + 2 * p - k) % s:
            continue
        din, dout, b = (int(v) for v in rng.integers(1, 9, size=3))
        b_p = int(rng.integers(1, b + 1))
        D, K = rand_case(rng, n, k, din, dout, b)
        spec = P.ConvSpec(n=n, k=k, d_in=din, d_out=dout, stride=s, pad=p)
        got = P.conv_lowered(P.Tensor4(D), P.Tensor4(K), spec, b_p=b_p, workers=1 + done % 3).values
        worst = max(worst, nrel(got, R.conv_direct(D, K, s, p)))
        done += 1
    assert worst < TOL, worst
