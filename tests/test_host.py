"""Host-side logic that needs no GPU: API validation (same messages as the
reference), network geometry and FLOP accounting, RNG streams, the group plan."""

import numpy as np
import pytest

import paper_1606_04487_b200 as P
from paper_1606_04487_b200 import nets
from oracle import refcnn as R


def test_convspec_validation_messages():
    with pytest.raises(ValueError, match="must be positive"):
        P.ConvSpec(n=0, k=1, d_in=1, d_out=1)
    with pytest.raises(ValueError, match="pad must be non-negative"):
        P.ConvSpec(n=4, k=1, d_in=1, d_out=1, pad=-1)
    with pytest.raises(ValueError, match="exceeds padded input"):
        P.ConvSpec(n=4, k=7, d_in=1, d_out=1)
    with pytest.raises(ValueError, match="not divisible by stride"):
        P.ConvSpec(n=8, k=3, d_in=1, d_out=1, stride=2)
    s = P.ConvSpec(n=227, k=11, d_in=3, d_out=96, stride=4)
    assert s.m == 55
    assert P.blowup_ratio(P.ConvSpec(n=4, k=3, d_in=1, d_out=1)) == 2.25
    assert P.blowup_ratio(P.ConvSpec(n=4, k=1, d_in=1, d_out=1)) == 1.0   # k=1: pure reshape


def test_tensor4_and_hyperparams():
    with pytest.raises(ValueError, match="expected 4 dims"):
        P.Tensor4(np.zeros((2, 2)))
    with pytest.raises(ValueError, match="non-finite"):
        P.Tensor4(np.full((1, 1, 2, 2), np.nan))
    t = P.Tensor4.from_flat((3, 3, 2, 1), np.arange(18.0))
    assert t.dims == (3, 3, 2, 1) and t.values.shape == (1, 2, 3, 3)
    for kw, msg in (({"eta": 0}, "eta must be positive"), ({"eta": 1, "mu": 1.0}, r"mu must be in"),
                    ({"eta": 1, "lam": -1}, "lambda must be"), ({"eta": 1, "b": 0}, "batch size")):
        with pytest.raises(ValueError, match=msg):
            P.Hyperparams(**kw)
    assert P.Hyperparams(eta=0.1).replace(mu=0.5).mu == 0.5
    with pytest.raises(ValueError, match="equal length"):
        P.SGDState(W=np.zeros(3), V=np.zeros(2))
    with pytest.raises(ValueError, match="max_steps"):
        P.StopRule(max_steps=0)


def test_smoothed_and_iterations_to_loss():
    losses = np.array([5.0, 4.0, 3.0, 2.0, 1.0])
    sm = P.smoothed(losses, window=2)
    assert np.allclose(sm, [5.0, 4.5, 3.5, 2.5, 1.5])
    tr = P.LossTrace(steps=np.arange(5), sim_times=np.arange(5.0), losses=losses,
                     final_state=P.SGDState.fresh(np.zeros(1)))
    assert P.iterations_to_loss(tr, 3.5, window=2) == 2
    assert P.iterations_to_loss(tr, 0.0, window=2) is None


def test_rng_streams_match_oracle():
    a = P.batch_stream(7, 3).integers(0, 100, size=10)
    b = R.batch_stream(7, 3).integers(0, 100, size=10)
    assert np.array_equal(a, b)
    assert P.child_seed(1, 2) == P.child_seed(1, 2) != P.child_seed(1, 3)


def test_execution_plan_and_models():
    plan = P.ExecutionPlan(N=8, g=4)
    assert plan.k == 2 and plan.staleness == 3
    assert [plan.group_of(r) for r in range(8)] == [0, 0, 1, 1, 2, 2, 3, 3]
    assert plan.group_ranks(2) == [4, 5]
    with pytest.raises(ValueError, match="does not divide"):
        P.ExecutionPlan(N=8, g=3)
    prof = P.PhaseProfile(T_cc=8.0, T_nc=0.1, t_fc=0.5)
    assert P.t_conv(2, prof) == 4.0
    assert P.he_predict(plan, prof) == max(0.5, (4.0 + 0.5) / 4)
    assert P.power_of_two_divisors(8) == [1, 2, 4, 8]
    assert [round(P.momentum_for_groups(g), 3) for g in (1, 2, 4, 8)] == [0.9, 0.4, 0.15, 0.025]


@pytest.mark.parametrize("name", list(nets.PRESETS))
def test_net_geometry_matches_oracle(name):
    net = nets.get(name)
    assert net.dim == R.param_count(net.to_dicts(), net.in_channels, net.in_size)


def test_caffenet_accounting():
    net = nets.caffenet()
    assert net.dim == 62_378_344
    assert abs(net.conv_flops_per_image() - 6.249e9) < 1e6   # 1.5997 TFLOP per 256
    g = net.geometry()
    assert [x.out_shape for x in g if x.layer.kind == "pool"] == [(96, 27, 27), (256, 13, 13), (256, 6, 6)]
    assert nets.cifar10_quick().geometry()[1].out_shape == (32, 16, 16)  # ceil-mode pooling
    assert abs(nets.vgg16().conv_flops_per_image() - 91.9e9) < 0.1e9


def test_netspec_validation():
    with pytest.raises(ValueError, match="end with a fully connected"):
        nets.NetSpec("x", 1, 8, (nets.Conv(4, 3),))
    with pytest.raises(ValueError, match="unknown network"):
        nets.get("resnet")
    with pytest.raises(ValueError, match="unknown pooling mode"):
        nets.Pool(2, mode="median")


def test_simconfig_validation():
    prof = P.PhaseProfile(T_cc=1.0, T_nc=0.0, t_fc=1.0)
    hp = P.Hyperparams(eta=0.1)
    with pytest.raises(ValueError, match="unknown service_mode"):
        P.SimConfig(plan=P.ExecutionPlan(2, 2), profile=prof, hp=hp, problem=None,
                    service_mode="x", max_updates=1)
    with pytest.raises(ValueError, match="need max_updates"):
        P.SimConfig(plan=P.ExecutionPlan(2, 2), profile=prof, hp=hp, problem=None)


@pytest.mark.parametrize("name", ["caffenet", "lenet", "cifar10_quick", "vgg16"])
def test_fc_head_split(name):
    """The merged-FC split: the head is the FC tail of the network and its
    parameters are the tail of the flat packing (problems.py:201-204)."""
    net = nets.get(name)
    head, off = nets.fc_head(net)
    assert all(L.kind in ("fc", "relu") for L in head.layers)
    assert head.dim == net.dim - off and head.classes == net.classes
    first_fc = next(g for g in net.geometry() if g.layer.kind == "fc")
    assert (head.in_channels, head.in_size, head.in_size) == first_fc.in_shape
    assert off == first_fc.param_offsets[0]


def test_bench_l2_note_classifies_working_sets():
    import importlib.util
    import os

    spec = importlib.util.spec_from_file_location(
        "bench", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    assert "> 126 MB L2" in bench.l2_note(nets.get("caffenet"), 256)
    assert "fits in L2" in bench.l2_note(nets.get("lenet"), 64)
