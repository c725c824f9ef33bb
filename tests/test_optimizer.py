"""Algorithm 1 (optimizer.py, SPEC.md auto-optimizer): selection semantics,
pruning, extension rounds, zero-momentum refinement, group halving control
flow and the checkpoint format -- with stubbed probe environments, as the
SPEC's examples prescribe."""

import numpy as np
import pytest

from paper_1606_04487_b200 import optimizer as O
from paper_1606_04487_b200.cluster import PhaseProfile
from paper_1606_04487_b200.sgd import SGDState

STATE = SGDState.fresh(np.zeros(3))


class StubEnv:
    """loss = f(g, mu, eta, seconds); records every probe."""

    def __init__(self, f, N=8, profile=PhaseProfile(T_cc=8.0, T_nc=0.0, t_fc=1.0)):
        self.f, self.N, self.profile, self.seed = f, N, profile, 0
        self.calls, self.sim_seconds = [], 0.0

    def run(self, state, g, mu, eta, secs, train=False):
        self.calls.append((g, mu, eta, secs))
        self.sim_seconds += secs
        loss = self.f(g, mu, eta, secs)
        return O.ProbeResult(state, loss, not np.isfinite(loss), 10)


GRID = O.GridSpec(probe_budget=1.0)


def test_single_point_grid_returns_it_after_one_probe():
    env = StubEnv(lambda *a: 1.0)
    assert O.grid_search(O.GridSpec(momentum_grid=(0.3,), probe_budget=1.0), STATE, 2, env, [0.01]) == (0.3, 0.01)
    assert len(env.calls) == 1


def test_selects_lowest_trailing_loss():
    env = StubEnv(lambda g, mu, eta, s: 0.5 if (mu, eta) == (0.6, 0.01) else 1.0)
    assert O.grid_search(GRID, STATE, 4, env, [0.01, 0.001]) == (0.6, 0.01)
    assert {(c[1], c[2]) for c in env.calls} == {(m, e) for m in GRID.momentum_grid for e in (0.01, 0.001)}


def test_pruning_skips_momenta_above_last_at_the_last_eta():
    env = StubEnv(lambda g, mu, eta, s: 1.0 + mu)
    O.grid_search(GRID, STATE, 4, env, [0.01, 0.001], last=(0.3, 0.01))
    probed = {(c[1], c[2]) for c in env.calls}
    assert (0.6, 0.01) not in probed and (0.9, 0.01) not in probed
    assert (0.9, 0.001) in probed and (0.3, 0.01) in probed


def test_close_calls_are_extended_until_a_clear_winner():
    # (0.3, .01) and (0.6, .01) are within 5% after one probe; (0.6, .01) pulls ahead later
    def f(g, mu, eta, s):
        if (mu, eta) == (0.3, 0.01):
            return 1.00
        if (mu, eta) == (0.6, 0.01):
            return 1.02 if s < 2.0 else 0.90
        return 2.0
    env = StubEnv(f)
    assert O.grid_search(GRID, STATE, 4, env, [0.01]) == (0.6, 0.01)
    assert max(c[3] for c in env.calls) == 2.0          # survivors ran a second, longer probe


def test_persistent_ties_go_to_lower_eta_then_lower_mu():
    env = StubEnv(lambda g, mu, eta, s: 1.0 if mu in (0.3, 0.6) else 3.0)
    assert O.grid_search(GRID, STATE, 4, env, [0.01, 0.001]) == (0.3, 0.001)


def test_all_diverged_is_an_error_with_diagnosis():
    env = StubEnv(lambda *a: float("inf"))
    with pytest.raises(RuntimeError, match="diverged"):
        O.grid_search(GRID, STATE, 2, env, [0.1])


@pytest.mark.parametrize("winner", [0.1, 0.0])
def test_refine_zero_momentum(winner):
    env = StubEnv(lambda g, mu, eta, s: 0.5 if mu == winner else 1.0)
    assert O.refine_zero_momentum(GRID, STATE, 4, env, 0.01) == winner


def test_halving_while_mu_star_is_zero():
    """SPEC: mu*=0 at g=8, mu*=0.3 at g=4 -> the epoch trains with g=4."""
    def f(g, mu, eta, s):
        best = 0.0 if g == 8 else 0.3
        return 0.5 if mu == best else 1.0
    env = StubEnv(f)
    _, log = O.optimize(None, env, GRID, O.EpochConfig(T=5.0, max_epochs=1),
                        start=(8, 0.9, 0.01, STATE))
    r = log.records[0]
    assert (r.g, r.mu) == (4, 0.3)
    assert 0.0 < r.probe_overhead_frac < 1.0
    trained = [c for c in env.calls if c[3] == 5.0]
    assert trained and trained[-1][0] == 4


def test_no_halving_when_mu_star_positive():
    env = StubEnv(lambda g, mu, eta, s: 0.5 if mu == 0.6 else 1.0)
    _, log = O.optimize(None, env, GRID, O.EpochConfig(T=5.0, max_epochs=2), start=(8, 0.9, 0.01, STATE))
    assert [r.g for r in log.records] == [8, 8] and all(r.mu == 0.6 for r in log.records)


def test_init_groups_is_the_smallest_saturating_count():
    # saturated iff t_conv(N/g) + t_fc < g t_fc (cluster.py:97-99); t_conv(k) = T_cc / k here
    assert O.init_groups(8, PhaseProfile(T_cc=2.0, T_nc=0.0, t_fc=1.0)) == (2, True)    # 0.5 + 1 < 2
    assert O.init_groups(8, PhaseProfile(T_cc=8.0, T_nc=0.0, t_fc=1.0)) == (8, False)   # never


def test_checkpoint_round_trip_and_corrupt_header(tmp_path):
    """SPEC.md:574 text format: lossless decimal round trip of binary64 and a
    header whose errors name the field."""
    rng = np.random.default_rng(0)
    W = rng.standard_normal(101) * 10.0 ** rng.integers(-300, 300, 101)
    W[:3] = [0.1, -0.0, 5e-324]
    ck = O.Checkpoint(W=W, V=rng.standard_normal(101), t=42, seed_cursor=2 ** 64 - 1)
    path = tmp_path / "a.omnickpt"
    O.save_checkpoint(ck, path)
    text = path.read_text().splitlines()
    assert text[0] == f"OMNISIM-CKPT v1 dim=101 t=42 seed_cursor={2 ** 64 - 1}"
    assert len(text) == 1 + 2 * 101 and text[1] == "0.1"
    back = O.load_checkpoint(path)
    assert np.array_equal(back.W, ck.W) and np.array_equal(back.V, ck.V)
    assert np.array_equal(np.signbit(back.W), np.signbit(ck.W))
    assert (back.t, back.seed_cursor) == (42, 2 ** 64 - 1)
    bad = tmp_path / "bad.omnickpt"
    bad.write_text("\n".join(["OMNISIM-CKPT v2 dim=101 t=42 seed_cursor=0"] + text[1:]) + "\n")
    with pytest.raises(ValueError, match="'version'"):
        O.load_checkpoint(bad)
    bad.write_text("\n".join(["OMNISIM-CKPT v1 dim=100 t=42 seed_cursor=0"] + text[1:]) + "\n")
    with pytest.raises(ValueError, match="'dim'"):
        O.load_checkpoint(bad)
    bad.write_text("\n".join(["OMNISIM-CKPT v1 dim=101 t=42"] + text[1:]) + "\n")
    with pytest.raises(ValueError, match="'seed_cursor'"):
        O.load_checkpoint(bad)


def test_training_epochs_advance_the_seed_cursor():
    """Probes of one round share the batch-stream seed (paired); every training
    epoch advances the cursor, so epochs do not replay the same batches."""
    env = O.SimEnv(None, N=8, profile=PhaseProfile(T_cc=1.0, T_nc=0.0, t_fc=0.1), b=4, seed=9)
    s0 = env.current_seed()
    env.seed_cursor += 1
    s1 = env.current_seed()
    env.seed_cursor += 1
    assert len({s0, s1, env.current_seed()}) == 3 and s0 == 9


def test_decision_log_csv(tmp_path):
    log = O.DecisionLog([O.DecisionRecord(0, 4, 0.3, 0.01, 0.1, 0.5, "c0")])
    log.write_csv(tmp_path / "log.csv")
    lines = (tmp_path / "log.csv").read_text().splitlines()
    assert lines[0] == "epoch,g,mu,eta,probe_overhead_frac,end_loss,checkpoint"
    assert lines[1].startswith("0,4,0.3,0.01,")
