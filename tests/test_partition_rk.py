"""Partition, exchange protocol, RK algebra, schedule and work model (host
logic; mirrors reference tests test_partition / test_rkcorrect / schedule)."""
import numpy as np
import pytest

from paper_2011_10570_b200.octree import OctKey, SfcOrdering, uniform_tree
from paper_2011_10570_b200.partition import (
    ExchangeError, ExchangePlan, PlanEntry, exchange, octant_weight, tree_weights, weighted_partition,
)
from paper_2011_10570_b200.perfmodel import WorkHistogram, estimate
from paper_2011_10570_b200.rkcorrect import (
    build_B, build_C, build_M, get_tableau, rk_step, stage_transfer_matrix,
)
from paper_2011_10570_b200.stepper import TimeLevelSchedule


class _T:
    def __init__(self, n):
        self.leaves = [None] * n


def test_weights():
    k = OctKey((0, 0), 3, 4)
    assert octant_weight(k, 3, "lts") == 1.0 and octant_weight(OctKey((0, 0), 4, 4), 2, "lts") == 4.0
    assert octant_weight(k, 1, "gts") == 1.0
    with pytest.raises(ValueError):
        octant_weight(k, 4, "lts")
    with pytest.raises(ValueError):
        octant_weight(k, 1, "xts")


def test_greedy_split_example_and_bound():
    pm = weighted_partition(_T(4), [1, 1, 2, 4], 2)
    assert pm.rank_ranges == [(0, 3), (3, 4)]
    rng = np.random.default_rng(0)
    for _ in range(200):
        n = int(rng.integers(1, 60))
        w = rng.choice([1.0, 2.0, 4.0, 8.0], size=n)
        R = int(rng.integers(1, 10))
        pm = weighted_partition(_T(n), w, R)
        assert pm.rank_ranges[0][0] == 0 and pm.rank_ranges[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(pm.rank_ranges, pm.rank_ranges[1:]))
        assert max(pm.rank_weights) <= w.sum() / R + w.max() + 1e-9
    with pytest.raises(ValueError):
        weighted_partition(_T(2), [1.0, 0.0], 2)
    with pytest.raises(ValueError):
        weighted_partition(_T(2), [1.0], 2)


def test_exchange_protocol():
    e = PlanEntry(0, 1, 5, 0, 3, 0, (1,))
    plan = ExchangePlan({(0, 1): [e]})
    assert exchange(plan, {(0, 1): [b"x"]}) == {(1, 0): [b"x"]}
    with pytest.raises(ExchangeError, match=r"\(0, 1\)"):
        exchange(plan, {})
    with pytest.raises(ExchangeError, match="oversized"):
        exchange(plan, {(0, 1): [b"a", b"b"]})
    with pytest.raises(ExchangeError, match="not in plan"):
        exchange(plan, {(0, 1): [b"a"], (1, 0): [b"b"]})


def test_tableaus_and_C():
    assert np.allclose(build_C(get_tableau("rk3")), [[1, 0, 0], [1, 0.5, 0], [1, 1, 1]])
    with pytest.raises(ValueError):
        get_tableau("rk9")
    assert np.allclose(build_B(0.0, 3), np.eye(3))


def test_M_frozen_rk2():
    M1, _, M2 = build_M(get_tableau("rk2"), 0.5, 1.0)
    assert np.allclose(M1, [[1, 0], [-1, 2]])
    assert np.allclose(M2, [[0, 1], [-0.5, 1.5]])
    with pytest.raises(ValueError):
        build_M(get_tableau("rk2"), 0.5, 1.5)


@pytest.mark.parametrize("name", ["rk2", "rk3", "rk4"])
def test_polynomial_forcing_exactness(name):
    tab = get_tableau(name)
    p = tab.stages
    g = lambda t: 1.0 + 2.0 * t  # stages expand exactly for forcing of degree <= 1  # noqa: E731
    t0, dtf, dtc = 0.3, 0.1, 0.2
    Kc = np.array([g(t0 + c * dtc) for c in tab.c])
    Kf = np.array([g(t0 + dtf + c * dtf) for c in tab.c])
    M = stage_transfer_matrix(tab, dtf, dtc, dtf)
    assert np.allclose(M @ Kc, Kf, atol=1e-12)


def test_rk3_decay_step_value():
    u, _ = rk_step(lambda t, u: -u, 1.0, 0.0, 0.1, get_tableau("rk3"))
    assert u == pytest.approx(0.9048333333333333, abs=1e-15)


def test_schedule():
    s = TimeLevelSchedule([4, 3, 2], l_max=4, l_min=2)
    assert s.slices_per_round == 4
    assert s.eligible(0) == [0, 1, 2] and s.eligible(1) == [0] and s.eligible(2) == [0, 1]
    assert s.phase(0) == 2 and s.phase(4) == 2 and s.phase(1) == 0 and s.phase(2) == 1
    assert [s.steps_per_round(b) for b in range(3)] == [4, 2, 1]


def test_work_model():
    est = estimate(WorkHistogram((1.0, 2.0)))
    assert est.w_lts == 1.0 * 2 + 2.0 and est.w_gts == 2 * 3.0 and est.speedup == 1.5 and est.bound == 3.0
    with pytest.raises(ValueError):
        WorkHistogram(())


def test_tree_weights():
    tree = uniform_tree(2, 3, 2, SfcOrdering("morton", 2, 3))
    assert np.all(tree_weights(tree, "lts") == 1.0) and np.all(tree_weights(tree, "gts") == 1.0)
