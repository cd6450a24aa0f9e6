"""Pin the CPU oracle (oracle/) against fixtures produced by the unmodified
reference (tests/golden/make_golden.py).  CPU only."""

import hashlib
import os

import numpy as np
import pytest

from conftest import golden
from oracle import oracle
from paper_1901_10084_b200 import instances


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make_oracle(oracle_lib, inst, kind="tiled", b=40, workers=1, reg_x=None, reg_f=None):
    return oracle_lib.OracleSolver(inst.n, inst.d_flat, inst.w_flat, inst.epsilon,
                                   reg_x=reg_x, reg_f=reg_f, kind=kind, b=b, workers=workers)


def test_config1_all_passes_bitwise(oracle_lib, config1_golden):
    g = config1_golden
    inst = instances.config_instance(1)
    assert sha(inst.d_flat) == str(g["dsha"]) and sha(inst.w_flat) == str(g["wsha"])
    o = make_oracle(oracle_lib, inst)
    for k in range(int(g["passes"])):
        st = o.run_pass()
        x, f = o.state()
        assert sha(x) == g["xsha"][k], k
        assert sha(f) == g["fsha"][k], k
        assert st.max_violation == g["viol"][k]
        assert st.primal_objective == pytest.approx(g["primal"][k], rel=1e-14, abs=1e-14)
        assert st.dual_objective == pytest.approx(g["dual"][k], rel=1e-14, abs=1e-14)
        keys, vals = o.duals()
        assert len(keys) == g["nnz"][k]
        assert sha(keys) == g["dkeys_sha"][k] and sha(vals) == g["dvals_sha"][k]
        assert sha(o.pair_duals()) == g["pd_sha"][k]
        assert st.steps == g["steps"][k]


@pytest.mark.parametrize("workers", [2, 5])
def test_worker_count_invariance(oracle_lib, workers):
    inst = instances.config_instance(1, n=61)
    a = make_oracle(oracle_lib, inst, b=8)
    c = make_oracle(oracle_lib, inst, b=8, workers=workers)
    for _ in range(6):
        sa, sc = a.run_pass(), c.run_pass()
        assert sa.max_violation == sc.max_violation
    assert np.array_equal(a.state()[0], c.state()[0])
    assert np.array_equal(a.state()[1], c.state()[1])
    ka, va = a.duals()
    kc, vc = c.duals()
    # same set of duals; the multi-worker order is per worker (core.py:218-227)
    assert np.array_equal(np.sort(ka), np.sort(kc))
    assert np.array_equal(va[np.argsort(ka)], vc[np.argsort(kc)])


SMALL = [(9, 2), (13, 3), (17, 5), (30, 8), (23, 4), (12, 1), (40, 40), (57, 16), (90, 40)]


@pytest.mark.parametrize("n,b", SMALL)
@pytest.mark.parametrize("wname", ["unit", "reg"])
def test_small_cases_bitwise(oracle_lib, small_golden, n, b, wname):
    g = small_golden
    tag = f"n{n}_b{b}_{wname}"
    inst = instances.random_instance(n, seed=1000 + n)
    rx = g[f"{tag}_regx"] if wname == "reg" else None
    rf = g[f"{tag}_regf"] if wname == "reg" else None
    o = make_oracle(oracle_lib, inst, b=b, reg_x=rx, reg_f=rf)
    for k in range(6):
        st = o.run_pass()
        assert st.max_violation == g[f"{tag}_viol"][k]
        assert st.primal_objective == pytest.approx(g[f"{tag}_primal"][k], rel=1e-13, abs=1e-13)
    x, f = o.state()
    assert np.array_equal(x, g[f"{tag}_x"])
    assert np.array_equal(f, g[f"{tag}_f"])
    keys, vals = o.duals()
    assert sha(keys) == str(g[f"{tag}_keysha"]) and sha(vals) == str(g[f"{tag}_valsha"])
    assert sha(o.pair_duals()) == str(g[f"{tag}_pdsha"])


def test_diagonal_bitwise(oracle_lib, small_golden):
    g = small_golden
    inst = instances.random_instance(14, seed=77)
    o = make_oracle(oracle_lib, inst, kind="diagonal")
    for _ in range(5):
        o.run_pass()
    x, f = o.state()
    assert np.array_equal(x, g["diag_n14_x"]) and np.array_equal(f, g["diag_n14_f"])
    keys, vals = o.duals()
    assert np.array_equal(keys, g["diag_n14_keys"]) and np.array_equal(vals, g["diag_n14_vals"])


@pytest.mark.parametrize("n", [4, 5, 6, 9])
def test_serial_bitwise_and_dense_algorithm1(oracle_lib, small_golden, n):
    g = small_golden
    inst = instances.random_instance(n, seed=100 * n)
    o = make_oracle(oracle_lib, inst, kind="serial")
    for _ in range(3):
        o.run_pass()
    x, f = o.state()
    assert np.array_equal(x, g[f"serial_n{n}_x"]) and np.array_equal(f, g[f"serial_n{n}_f"])
    keys, vals = o.duals()
    assert np.array_equal(keys, g[f"serial_n{n}_keys"])
    assert np.array_equal(vals, g[f"serial_n{n}_vals"])
    if n <= 6:  # reference tests' dense Algorithm 1 (tests/reference.py:57-75)
        assert np.max(np.abs(np.concatenate([x, f]) - g[f"dense_n{n}_v"])) <= 1e-10


@pytest.mark.parametrize("n", [7, 31])
def test_max_violation_scan(oracle_lib, small_golden, n):
    g = small_golden
    inst = instances.random_instance(n, seed=n)
    v = oracle_lib.max_violation(g[f"scan_n{n}_x"], g[f"scan_n{n}_f"], inst.d_flat, n)
    assert v == float(g[f"scan_n{n}_viol"])


@pytest.mark.parametrize("kind,b", [("tiled", 3), ("tiled", 5), ("diagonal", 1), ("serial", 40)])
def test_python_restatement_matches_c(oracle_lib, kind, b):
    n = 11
    inst = instances.random_instance(n, seed=5)
    rng = np.random.default_rng(3)
    rx = rng.uniform(0.5, 2.0, inst.npairs)
    rf = rng.uniform(0.5, 2.0, inst.npairs)
    o = make_oracle(oracle_lib, inst, kind=kind, b=b, reg_x=rx, reg_f=rf)
    x = np.zeros(inst.npairs)
    f = -inst.w_flat / (inst.epsilon * rf)
    duals, pd = {}, np.zeros((inst.npairs, 2))
    for _ in range(4):
        st = o.run_pass()
        viol, duals = oracle_lib.py_pass(n, inst.epsilon, x, f, inst.d_flat, 1.0 / rx, 1.0 / rf,
                                         duals, pd, kind=kind, b=b)
        assert viol == st.max_violation
    ox, of = o.state()
    assert np.array_equal(ox, x) and np.array_equal(of, f)
    keys, vals = o.duals()
    assert dict(zip(keys.tolist(), vals.tolist())) == duals
    assert np.array_equal(o.pair_duals(), pd)


def test_config2_first_passes(oracle_lib):
    g = golden("config2_n1000_b40_p4")
    inst = instances.config_instance(2)
    assert sha(inst.d_flat) == str(g["dsha"])
    o = make_oracle(oracle_lib, inst, workers=8)
    for k in range(int(g["passes"])):
        st = o.run_pass()
        x, _ = o.state()
        assert sha(x) == g["xsha"][k]
        assert st.max_violation == g["viol"][k]
        assert len(o.duals()[0]) == g["nnz"][k]
    x, f = o.state()
    idx = g["sample_idx"]
    assert np.array_equal(x[idx], g["sample_x_final"])
    assert np.array_equal(f[idx], g["sample_f_final"])


def test_schedule_export_matches_python(oracle_lib):
    from paper_1901_10084_b200 import schedule
    for n, b in [(10, 3), (57, 16), (100, 40), (33, 1)]:
        inst = instances.random_instance(n, seed=1)
        o = make_oracle(oracle_lib, inst, b=b)
        rn, xz = o.schedule()
        rounds = schedule.tiled_rounds(n, b)
        assert list(rn) == [len(r.units) for r in rounds]
        assert [tuple(t) for t in xz] == [(u.x, u.z) for r in rounds for u in r.units]


def _aty_cases():
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "aty.npz"))
    return z, [(p, int(z[p + "_n"])) for p in ("r", "c")]


def test_oracle_accumulate_aty_matches_reference_golden():
    """Both restatements of core.accumulate_aty (core.py:285-293) equal the
    reference's own output bit for bit (tests/golden/make_aty_golden.py)."""
    z, cases = _aty_cases()
    for p, n in cases:
        args = (n, z[p + "_keys"], z[p + "_vals"], z[p + "_pd"], z[p + "_c"])
        g = oracle.accumulate_aty_np(*args)
        assert np.array_equal(g, z[p + "_g"]), p
        if p == "r":
            assert np.array_equal(oracle.accumulate_aty_loop(*args), z[p + "_g"])
