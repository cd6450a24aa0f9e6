"""Host-side domain model (mirror of the reference's core.py).  CPU only."""

import json

import numpy as np
import pytest
from hypothesis import given, strategies as st

from oracle import oracle
from paper_1901_10084_b200 import core, instances
from paper_1901_10084_b200.core import (ConstraintKey, DualStore, Kind, PassStats, PrimalState,
                                         ProblemInstance)


def test_pair_index_matches_triu_order():
    for n in (3, 5, 9):
        iu = np.triu_indices(n, 1)
        for pos, (i, j) in enumerate(zip(*iu)):
            assert core.pair_index(n, int(i), int(j)) == pos
    for bad in ((3, 3), (4, 2), (0, 5)):
        with pytest.raises(ValueError):
            core.pair_index(5, *bad)


def test_constraint_count():
    for n in range(3, 12):
        assert core.constraint_count(n, metric_only=True) == 3 * (n * (n - 1) * (n - 2) // 6)
        assert core.constraint_count(n) == 3 * (n * (n - 1) * (n - 2) // 6) + n * (n - 1)
    with pytest.raises(ValueError):
        core.constraint_count(2)
    assert f"{core.constraint_count(17903, metric_only=True):.1e}" == "2.9e+12"


@given(st.integers(4, 200), st.data())
def test_key_roundtrip(n, data):
    i = data.draw(st.integers(0, n - 3))
    j = data.draw(st.integers(i + 1, n - 2))
    k = data.draw(st.integers(j + 1, n - 1))
    kind = data.draw(st.sampled_from(core.METRIC_KINDS))
    key = ConstraintKey(kind, i, j, k)
    assert ConstraintKey.decode(key.encode(n), n) == key
    ii, jj, kk, kd = core.decode_keys(np.array([key.encode(n)]), n)
    assert (ii[0], jj[0], kk[0], kd[0]) == (i, j, k, int(kind))


def test_key_validation():
    with pytest.raises(ValueError):
        ConstraintKey(Kind.METRIC_IJ, 2, 1, 3)
    with pytest.raises(ValueError):
        ConstraintKey(Kind.PAIR_UPPER, 1, 2, 3)


def test_instance_validation_and_flat():
    n = 4
    D, Wt = np.zeros((n, n)), np.ones((n, n))
    ProblemInstance(n, D, Wt)
    with pytest.raises(ValueError):
        ProblemInstance(2, np.zeros((2, 2)), np.ones((2, 2)))
    bad = D.copy()
    bad[0, 1] = 1.0
    with pytest.raises(ValueError):
        ProblemInstance(n, bad, Wt)
    with pytest.raises(ValueError):
        ProblemInstance(n, D, Wt, epsilon=0.0)
    with pytest.raises(ValueError):
        ProblemInstance(n, D, Wt * 0.0)
    inst = instances.random_instance(7, seed=3)
    flat = ProblemInstance.from_flat(7, inst.d_flat, inst.w_flat, epsilon=inst.epsilon)
    assert np.array_equal(flat.D, inst.D) and np.array_equal(flat.Wt[np.triu_indices(7, 1)], inst.w_flat)
    assert inst.rhs(ConstraintKey(Kind.PAIR_LOWER, 1, 3)) == -inst.D[1, 3]


def test_primal_state_orientation():
    s = PrimalState(5)
    s.set_x(3, 1, 2.5)
    assert s.get_x(1, 3) == 2.5 and s.get_x(2, 2) == 0.0
    X = s.X()
    assert np.array_equal(X, X.T) and X[1, 3] == 2.5
    with pytest.raises(ValueError):
        s.set_x(2, 2, 1.0)


def dense_rows(n, d):
    """Dense constraint rows in serial order (an independent restatement)."""
    m = n * (n - 1) // 2
    rows = []
    for (i, j, k) in __import__("itertools").combinations(range(n), 3):
        p = [core.pair_index(n, *pr) for pr in ((i, j), (i, k), (j, k))]
        for plus, m1, m2 in ((p[0], p[1], p[2]), (p[1], p[0], p[2]), (p[2], p[0], p[1])):
            a = np.zeros(2 * m)
            a[plus], a[m1], a[m2] = 1, -1, -1
            rows.append(a)
    for q in range(m):
        a = np.zeros(2 * m); a[q], a[m + q] = 1, -1
        rows.append(a)
        a = np.zeros(2 * m); a[q], a[m + q] = -1, -1
        rows.append(a)
    return rows


def test_accumulate_aty_matches_dense():
    n = 6
    inst = instances.random_instance(n, seed=2)
    rng = np.random.default_rng(0)
    d = DualStore(n, 2)
    keys = [ConstraintKey(Kind(rng.integers(3)), *sorted(rng.choice(n, 3, replace=False))) for _ in range(8)]
    codes = np.unique([k.encode(n) for k in keys])
    d.keys = [codes[:3], codes[3:]]
    vals = rng.uniform(0.1, 1.0, len(codes))
    d.vals = [vals[:3], vals[3:]]
    d.pair_duals = rng.uniform(0, 1, (inst.npairs, 2)) * (rng.uniform(size=(inst.npairs, 2)) < 0.5)
    k_all, v_all = d.metric_arrays()
    g = oracle.accumulate_aty_np(n, k_all, v_all, d.pair_duals, inst.c_vector())
    assert np.array_equal(g, oracle.accumulate_aty_loop(n, k_all, v_all, d.pair_duals, inst.c_vector()))
    rows = dense_rows(n, inst.d_flat)
    ntrip = n * (n - 1) * (n - 2) // 6
    y = np.zeros(len(rows))
    for c, v in zip(codes, vals):
        key = ConstraintKey.decode(int(c), n)
        order = list(__import__("itertools").combinations(range(n), 3)).index((key.i, key.j, key.k))
        y[3 * order + int(key.kind)] = v
    y[3 * ntrip::2] = d.pair_duals[:, 0]
    y[3 * ntrip + 1::2] = d.pair_duals[:, 1]
    expect = inst.c_vector() + np.array(rows).T @ y
    assert np.allclose(g, expect, atol=1e-12)


def test_objectives_match_dense_formula():
    inst = instances.random_instance(6, seed=123)
    rng = np.random.default_rng(0)
    s = PrimalState(6, rng.normal(size=inst.npairs), rng.normal(size=inst.npairs))
    v = s.v()
    expect = inst.c_vector() @ v + 0.5 * inst.epsilon * v @ v
    assert core.primal_objective(inst, s) == pytest.approx(expect, rel=1e-12)


def test_dual_store_items_and_stats_json():
    d = DualStore(5, 1)
    d.keys = [np.array([ConstraintKey(Kind.METRIC_IK, 0, 2, 4).encode(5)])]
    d.vals = [np.array([0.25])]
    d.pair_duals[3] = (0.5, 0.0)
    items = list(d.items())
    assert items[0] == (ConstraintKey(Kind.METRIC_IK, 0, 2, 4), 0.25)
    assert items[1][0].kind == Kind.PAIR_UPPER and items[1][1] == 0.5
    assert d.nnz() == 1
    s = PassStats(1, 2.0, 1.0, 1.0, 0.1, 0.5, steps=9)
    p = json.loads(s.to_json())
    assert "steps" not in p and p["pass_index"] == 1
