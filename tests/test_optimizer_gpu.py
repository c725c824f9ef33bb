"""Algorithm 1 end to end on the device-resident simulator (TinyCNN)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1606_04487_b200 as P  # noqa: E402
from paper_1606_04487_b200 import optimizer as O  # noqa: E402
from paper_1606_04487_b200.problems import TinyCNNProblem  # noqa: E402


def test_algorithm1_runs_and_keeps_its_invariants(tmp_path):
    # the PhaseProfile measured on B200 by tools/async_he.py (CaffeNet, seconds)
    prob = TinyCNNProblem(8, 4, seed=3, n_examples=64)
    env = O.SimEnv(prob, N=8, profile=P.PhaseProfile(T_cc=3.43e-3, T_nc=0.49e-3, t_fc=0.81e-3),
                   b=16, seed=5, loss_sample_interval=4)
    grid = O.GridSpec(probe_budget=0.02)
    state, log = O.optimize(prob, env, grid, O.EpochConfig(T=0.2, max_epochs=2),
                            checkpoint_dir=str(tmp_path))
    gs = [r.g for r in log.records]
    assert all(a >= b for a, b in zip(gs, gs[1:]))                   # monotone halving
    assert all(r.mu != 0.0 or r.g == 1 for r in log.records)        # Algorithm 1 postcondition
    assert all(0.0 < r.probe_overhead_frac < 1.0 for r in log.records)
    ck = O.load_checkpoint(log.records[-1].checkpoint)
    assert np.array_equal(ck.W, np.asarray(state.W)) and ck.t == state.t
    assert np.isfinite(log.records[-1].end_loss)
    assert log.records[-1].end_loss < 0.8 * prob.full_loss(prob.initial_weights())
    log.write_csv(tmp_path / "decisions.csv")
