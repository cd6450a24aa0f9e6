"""Schedule and the device's execution order: partition, independence, and
the two ordering facts the CUDA kernel relies on (CPU only):

1. sweeping a tile by levels L = i+j+k is a linear extension of the
   reference's cube order restricted to conflicting triplets;
2. every conflict is ordered along the (i,k) lattice -- the later triplet's
   (i,k) is reachable from the earlier one's by +1 steps in i or k, one level
   per step -- so per-warp progress counters replace CTA barriers.
"""

import itertools

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from paper_1901_10084_b200 import schedule


@pytest.mark.parametrize("n,b", [(3, 1), (7, 2), (12, 3), (20, 5), (33, 8), (50, 16), (61, 40)])
def test_partition_and_independence(n, b):
    rounds = schedule.tiled_rounds(n, b)
    assert schedule.verify_partition(rounds, n)
    assert schedule.verify_independence(rounds, n)


def test_diagonal_equals_tiled_b1():
    for n in (5, 9, 14):
        d = schedule.diagonal_rounds(n)
        t = schedule.tiled_rounds(n, 1)
        assert [[(u.i, u.k) for u in r.units] for r in d] == [[(u.x, u.z) for u in r.units] for r in t]


def conflicts(a, b):
    return len(set(a) & set(b)) >= 2


@pytest.mark.parametrize("n,b", [(12, 3), (17, 5), (30, 8), (45, 16)])
def test_level_order_is_linear_extension(n, b):
    for rnd in schedule.tiled_rounds(n, b):
        for tile in rnd.units:
            ref = list(schedule.tile_triplets(tile, n))
            pos = {t: p for p, t in enumerate(ref)}
            dev = schedule.tile_level_order(tile, n)
            dpos = {t: p for p, t in enumerate(dev)}
            assert sorted(ref) == sorted(dev)
            for t1, t2 in itertools.combinations(ref, 2):
                if conflicts(t1, t2):
                    assert (pos[t1] < pos[t2]) == (dpos[t1] < dpos[t2]), (tile, t1, t2)
                    assert sum(t1) != sum(t2)


@pytest.mark.parametrize("n,b", [(12, 3), (19, 5), (40, 12), (45, 16)])
def test_conflicts_ordered_along_lattice(n, b):
    for rnd in schedule.tiled_rounds(n, b):
        for tile in rnd.units:
            ref = list(schedule.tile_triplets(tile, n))
            for p, q in itertools.combinations(range(len(ref)), 2):
                t1, t2 = ref[p], ref[q]  # reference visits t1 first
                if not conflicts(t1, t2):
                    continue
                (i1, _, k1), (i2, _, k2) = t1, t2
                dl = sum(t2) - sum(t1)
                assert i2 >= i1 and k2 >= k1 and dl >= (i2 - i1) + (k2 - k1), (t1, t2)


@pytest.mark.parametrize("n,b", [(20, 3), (33, 5), (57, 16), (100, 40), (90, 40), (41, 1)])
def test_touched_pairs_matches_enumeration(n, b):
    assert schedule.touched_pairs(n, b) == schedule.touched_pairs_brute(n, b)


def test_touched_pairs_survey_values():
    # exact T_x at b = 40
    assert schedule.touched_pairs(100, 40) == 13643
    assert schedule.touched_pairs(1000, 40) == 8814025


def test_critical_levels_survey_value():
    assert schedule.critical_levels(1000, 40) == 28792  # SURVEY.md A.3 barrier depth


@settings(max_examples=40, deadline=None)
@given(st.integers(3, 60), st.integers(1, 48))
def test_tile_level_ranges(n, b):
    for rnd in schedule.tiled_rounds(n, b):
        for t in rnd.units:
            lo, hi = t.levels()
            sums = [sum(x) for x in schedule.tile_triplets(t, n)]
            assert min(sums) == lo and max(sums) == hi


@pytest.mark.parametrize("n,c", [(11, 3), (17, 4), (20, 5), (23, 8)])
def test_cube_order_equals_serial(n, c):
    """The cube-blocked wavefront (cube levels, then L levels inside a cube)
    reproduces schedule_kind="serial" bit for bit, with
    non-identity W and stored duals (3 passes)."""
    import numpy as np
    from oracle import oracle as orc
    rng = np.random.default_rng(n * 31 + c)
    m = n * (n - 1) // 2
    d = rng.integers(0, 2, m).astype(float)
    winvx = 1.0 / rng.uniform(0.5, 2.0, m)
    winvf = 1.0 / rng.uniform(0.5, 2.0, m)
    eps = 0.3
    states = []
    for kind in ("serial", "cube"):
        x = np.zeros(m)
        f = -np.ones(m) / eps
        duals, pd = {}, np.zeros((m, 2))
        for _ in range(3):
            _, duals = orc.py_pass(n, eps, x, f, d, winvx, winvf, duals, pd, kind=kind, b=c)
        states.append((x.copy(), f.copy(), sorted(duals.items())))
    assert np.array_equal(states[0][0], states[1][0])
    assert np.array_equal(states[0][1], states[1][1])
    assert states[0][2] == states[1][2]


def test_worker_of_keys_matches_round_positions():
    """The per-worker DualStore layout of a workers = p reference run: a key's
    worker is (position of its tile in its round + 1) mod p (schedule.py:79-80,
    solver.py:86-91) -- computed from the key alone."""
    import numpy as np
    from paper_1901_10084_b200 import core
    from paper_1901_10084_b200.solver import worker_of_keys
    for n, b, p in [(23, 4, 3), (41, 5, 8), (30, 40, 2), (19, 1, 4)]:
        rounds = schedule.tiled_rounds(n, b) if b > 1 else schedule.diagonal_rounds(n)
        for rnd in rounds:
            for pos, unit in enumerate(rnd.units):
                trips = list(schedule.unit_triplets(unit, n))
                keys = np.array([core.ConstraintKey(core.Kind.METRIC_IJ, i, j, k).encode(n)
                                 for (i, j, k) in trips], dtype=np.int64)
                assert set(worker_of_keys(keys, n, b, p).tolist()) == {rnd.worker_of(pos, p)}
