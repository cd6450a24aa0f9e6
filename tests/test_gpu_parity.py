"""GPU parity: the CUDA path (through the C ABI) against reference-generated
fixtures and the CPU oracle.  x, f and all duals must be BITWISE equal
(integer/fp64 replay of the reference order); objectives within 1e-12 rel."""

import hashlib

import numpy as np
import pytest

from conftest import golden
from paper_1901_10084_b200 import instances
from paper_1901_10084_b200.solver import DeviceSession

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_config1_every_pass_bitwise(config1_golden):
    g = config1_golden
    inst = instances.config_instance(1)
    sess = DeviceSession(inst, "tiled", 40)
    for k in range(int(g["passes"])):
        st = sess.run(1)[0]
        x, f = sess.state()
        assert sha(x) == g["xsha"][k], f"x differs after pass {k + 1}"
        assert sha(f) == g["fsha"][k], f"f differs after pass {k + 1}"
        assert st.max_violation == g["viol"][k]
        assert st.nnz_metric == g["nnz"][k]
        assert st.primal_objective == pytest.approx(g["primal"][k], rel=1e-12, abs=1e-12)
        assert st.dual_objective == pytest.approx(g["dual"][k], rel=1e-12, abs=1e-12)
        assert st.steps == g["steps"][k]
        if k + 1 in (2, 3, 50):
            assert np.array_equal(x, g[f"x_{k + 1}"])
    keys, vals, pd = sess.duals()
    assert sha(keys) == g["dkeys_sha"][-1] and sha(vals) == g["dvals_sha"][-1]
    assert sha(pd) == g["pd_sha"][-1]


SMALL = [(9, 2), (13, 3), (17, 5), (30, 8), (23, 4), (12, 1), (40, 40), (57, 16), (90, 40)]


@pytest.mark.parametrize("n,b", SMALL)
@pytest.mark.parametrize("wname", ["unit", "reg"])
def test_small_cases_bitwise(small_golden, n, b, wname):
    g = small_golden
    tag = f"n{n}_b{b}_{wname}"
    inst = instances.random_instance(n, seed=1000 + n)
    if wname == "reg":
        inst.reg_x = g[f"{tag}_regx"]
        inst.reg_f = g[f"{tag}_regf"]
    sess = DeviceSession(inst, "tiled", b)
    for k in range(6):
        st = sess.run(1)[0]
        assert st.max_violation == g[f"{tag}_viol"][k]
        assert st.primal_objective == pytest.approx(g[f"{tag}_primal"][k], rel=1e-12, abs=1e-12)
        assert st.dual_objective == pytest.approx(g[f"{tag}_dual"][k], rel=1e-12, abs=1e-12)
    x, f = sess.state()
    assert np.array_equal(x, g[f"{tag}_x"])
    assert np.array_equal(f, g[f"{tag}_f"])
    keys, vals, pd = sess.duals()
    assert sha(keys) == str(g[f"{tag}_keysha"]) and sha(vals) == str(g[f"{tag}_valsha"])
    assert sha(pd) == str(g[f"{tag}_pdsha"])


def test_diagonal_bitwise(small_golden):
    g = small_golden
    inst = instances.random_instance(14, seed=77)
    sess = DeviceSession(inst, "diagonal", 40)
    sess.run(5)
    x, f = sess.state()
    assert np.array_equal(x, g["diag_n14_x"]) and np.array_equal(f, g["diag_n14_f"])
    keys, vals, _ = sess.duals()
    assert np.array_equal(keys, g["diag_n14_keys"]) and np.array_equal(vals, g["diag_n14_vals"])


def test_config2_first_passes_bitwise():
    g = golden("config2_n1000_b40_p4")
    inst = instances.config_instance(2)
    sess = DeviceSession(inst, "tiled", 40)
    for k in range(int(g["passes"])):
        st = sess.run(1)[0]
        x, _ = sess.state()
        assert sha(x) == g["xsha"][k], k
        assert st.max_violation == g["viol"][k]
        assert st.nnz_metric == g["nnz"][k]
    x, f = sess.state()
    assert np.array_equal(x[g["sample_idx"]], g["sample_x_final"])
    assert np.array_equal(f[g["sample_idx"]], g["sample_f_final"])


@pytest.mark.parametrize("config,n,b,passes", [(1, 100, 40, 12), (3, 300, 40, 6), (4, 200, 16, 6),
                                               (5, 260, 48, 5), (2, 240, 32, 5), (1, 150, 24, 8)])
def test_against_oracle(oracle_lib, config, n, b, passes):
    inst = instances.config_instance(config, n=n)
    sess = DeviceSession(inst, "tiled", b)
    ref = oracle_lib.OracleSolver(inst.n, inst.d_flat, inst.w_flat, inst.epsilon, b=b, workers=4)
    for _ in range(passes):
        st = sess.run(1)[0]
        rs = ref.run_pass()
        assert st.max_violation == rs.max_violation
        assert st.primal_objective == pytest.approx(rs.primal_objective, rel=1e-12)
    x, f = sess.state()
    rx, rf = ref.state()
    assert np.array_equal(x, rx) and np.array_equal(f, rf)
    keys, vals, pd = sess.duals()
    rk, rv = ref.duals()  # 4 workers: concatenated per worker (core.py:218-236)
    o1, o2 = np.argsort(keys), np.argsort(rk)
    assert np.array_equal(keys[o1], rk[o2]) and np.array_equal(vals[o1], rv[o2])
    assert np.array_equal(pd, ref.pair_duals())


def test_dual_import_resumes_oracle_run(oracle_lib):
    """mp_set_state / mp_set_duals: continue a CPU run on the device."""
    inst = instances.config_instance(1, n=80)
    ref = oracle_lib.OracleSolver(inst.n, inst.d_flat, inst.w_flat, inst.epsilon, b=16)
    for _ in range(3):
        ref.run_pass()
    sess = DeviceSession(inst, "tiled", 16)
    x, f = ref.state()
    keys, vals = ref.duals()
    sess.set_state(x, f)
    sess.set_duals(keys, vals, ref.pair_duals())
    for _ in range(3):
        st = sess.run(1)[0]
        rs = ref.run_pass()
        assert st.max_violation == rs.max_violation
    assert np.array_equal(sess.state()[0], ref.state()[0])
    k2, v2, _ = sess.duals()
    rk, rv = ref.duals()
    assert np.array_equal(k2, rk) and np.array_equal(v2, rv)


@pytest.mark.parametrize("n", [7, 31])
def test_exact_violation_scan(small_golden, n):
    from paper_1901_10084_b200 import core
    g = small_golden
    inst = instances.random_instance(n, seed=n)
    st = core.PrimalState(n, g[f"scan_n{n}_x"], g[f"scan_n{n}_f"])
    assert core.max_violation(inst, st) == float(g[f"scan_n{n}_viol"])


def test_session_violation_scan_matches_oracle(oracle_lib):
    inst = instances.config_instance(1)
    sess = DeviceSession(inst, "tiled", 40)
    sess.run(5)
    x, f = sess.state()
    assert sess.max_violation() == oracle_lib.max_violation(x, f, inst.d_flat, inst.n)


@pytest.mark.parametrize("n", [4, 5, 6, 9])
def test_serial_schedule_bitwise(small_golden, n):
    """schedule_kind='serial' (_kernels.py:135-183) on the device."""
    g = small_golden
    inst = instances.random_instance(n, seed=100 * n)
    sess = DeviceSession(inst, "serial", 40)
    sess.run(3)
    x, f = sess.state()
    assert np.array_equal(x, g[f"serial_n{n}_x"]) and np.array_equal(f, g[f"serial_n{n}_f"])
    keys, vals, _ = sess.duals()
    assert np.array_equal(keys, g[f"serial_n{n}_keys"]) and np.array_equal(vals, g[f"serial_n{n}_vals"])
    if n <= 6:  # the reference tests' dense Algorithm 1 (tests/reference.py:57-75)
        assert np.max(np.abs(np.concatenate([x, f]) - g[f"dense_n{n}_v"])) <= 1e-10


@pytest.mark.parametrize("n,reg", [(40, False), (77, True), (150, False), (333, False), (260, True)])
def test_serial_against_oracle(oracle_lib, n, reg):
    inst = instances.config_instance(1, n=n)
    rx = rf = None
    if reg:
        rng = np.random.default_rng(n)
        rx = rng.uniform(0.5, 2.0, inst.npairs)
        rf = rng.uniform(0.5, 2.0, inst.npairs)
        inst.reg_x, inst.reg_f = rx, rf
    sess = DeviceSession(inst, "serial", 40)
    ref = oracle_lib.OracleSolver(inst.n, inst.d_flat, inst.w_flat, inst.epsilon, reg_x=rx,
                                  reg_f=rf, kind="serial")
    for _ in range(5):
        st = sess.run(1)[0]
        rs = ref.run_pass()
        assert st.max_violation == rs.max_violation
    x, f = sess.state()
    assert np.array_equal(x, ref.state()[0]) and np.array_equal(f, ref.state()[1])
    keys, vals, _ = sess.duals()
    rk, rv = ref.duals()
    assert np.array_equal(keys, rk) and np.array_equal(vals, rv)
    # import the oracle's duals and state, continue both: still identical
    sess2 = DeviceSession(inst, "serial", 40)
    sess2.set_state(*ref.state())
    sess2.set_duals(rk, rv, ref.pair_duals())
    sess2.run(2)
    ref.run_pass()
    ref.run_pass()
    assert np.array_equal(sess2.state()[0], ref.state()[0])


@pytest.mark.parametrize("divisor", [0.2, 0.1, 0.7, 0.3, 0.5, 3.0, 1.0 / 7.0, 0.123456789])
def test_fast_division_is_ieee(divisor):
    """div_rn (Markstein step with RN(1/b)) equals IEEE division bit for bit."""
    import ctypes
    from paper_1901_10084_b200 import _native
    bad = np.zeros(1, dtype=np.int64)
    _native.check(_native.load().mp_check_division(divisor, 20_000_000, 12345, _native.iptr(bad)),
                  "mp_check_division")
    assert bad[0] == 0


@pytest.mark.parametrize("cluster,slots", [(1, None), (2, None), (3, None), (5, None), (8, None),
                                           (4, 2), (8, 2), (6, 3)])
@pytest.mark.parametrize("general_w", [False, True])
def test_cluster_shapes_bitwise(oracle_lib, knobs, cluster, slots, general_w):
    """Every launch shape -- C CTAs per tile (row bands, DSMEM forwarding of
    the replicated WK/RK), S slots per thread -- follows the reference order
    bit for bit (MP_CLUSTER caps C; MP_SLOTS raises S)."""
    knobs.setenv("MP_CLUSTER", str(cluster))
    if slots:
        knobs.setenv("MP_SLOTS", str(slots))
    inst = instances.config_instance(1, n=180)
    rx = rf = None
    if general_w:
        rng = np.random.default_rng(5)
        rx = rng.uniform(0.5, 2.0, inst.npairs)
        rf = rng.uniform(0.5, 2.0, inst.npairs)
        inst.reg_x, inst.reg_f = rx, rf
    sess = DeviceSession(inst, "tiled", 40)
    ref = oracle_lib.OracleSolver(inst.n, inst.d_flat, inst.w_flat, inst.epsilon, reg_x=rx, reg_f=rf,
                                  b=40, workers=4)
    for _ in range(4):
        st = sess.run(1)[0]
        rs = ref.run_pass()
        assert st.max_violation == rs.max_violation
    x, f = sess.state()
    assert np.array_equal(x, ref.state()[0]) and np.array_equal(f, ref.state()[1])
    keys, vals, _ = sess.duals()
    rk, rv = ref.duals()
    o1, o2 = np.argsort(keys), np.argsort(rk)
    assert np.array_equal(keys[o1], rk[o2]) and np.array_equal(vals[o1], rv[o2])
    sess.close()


@pytest.mark.parametrize("kind,cluster", [("tiled", 8), ("tiled", 1), ("serial", 1)])
def test_dual_pool_overflow_rolls_back(oracle_lib, knobs, kind, cluster):
    """A dual pool far too small: every pass overflows at first, is rolled
    back from its snapshot and redone with a larger pool -- the trajectory
    is unchanged (solver.run_pass semantics, bitwise vs the oracle)."""
    knobs.setenv("MP_POOL_CAP0", "2")
    knobs.setenv("MP_CLUSTER", str(cluster))
    inst = instances.config_instance(1, n=120)
    sess = DeviceSession(inst, kind, 40)
    ref = oracle_lib.OracleSolver(inst.n, inst.d_flat, inst.w_flat, inst.epsilon, kind=kind, b=40)
    for _ in range(4):
        st = sess.run(1)[0]
        rs = ref.run_pass()
        assert st.max_violation == rs.max_violation
        assert st.nnz_metric == len(ref.duals()[0])
    assert np.array_equal(sess.state()[0], ref.state()[0])
    keys, vals, _ = sess.duals()
    rk, rv = ref.duals()
    o1, o2 = np.argsort(keys), np.argsort(rk)
    assert np.array_equal(keys[o1], rk[o2]) and np.array_equal(vals[o1], rv[o2])
    sess.close()


@pytest.mark.parametrize("n", [180, 181])  # even n: TMA boxes for WK; odd n: odd klo, element copies
@pytest.mark.parametrize("cluster", [8, 4, 1])
@pytest.mark.parametrize("env", [{}, {"MP_WR_PITCH_W": "1", "MP_WK_PITCH_B": "1"}, {"MP_NO_TMA": "1"}])
def test_ring_staging_variants_bitwise(oracle_lib, knobs, n, cluster, env):
    """Every way of staging the j-rings -- WK as 2-D TMA boxes (plain or
    padded row pitch, box or 16-byte write-back) or element by element,
    padded or plain WR pitch -- gives the reference trajectory bit for bit."""
    knobs.setenv("MP_CLUSTER", str(cluster))
    for k, v in env.items():
        knobs.setenv(k, v)
    inst = instances.config_instance(2, n=n)
    sess = DeviceSession(inst, "tiled", 40)
    ref = oracle_lib.OracleSolver(inst.n, inst.d_flat, inst.w_flat, inst.epsilon, b=40, workers=4)
    for _ in range(4):
        st = sess.run(1)[0]
        rs = ref.run_pass()
        assert st.max_violation == rs.max_violation
    x, f = sess.state()
    assert np.array_equal(x, ref.state()[0]) and np.array_equal(f, ref.state()[1])
    keys, vals, _ = sess.duals()
    rk, rv = ref.duals()
    o1, o2 = np.argsort(keys), np.argsort(rk)
    assert np.array_equal(keys[o1], rk[o2]) and np.array_equal(vals[o1], rv[o2])
    sess.close()
