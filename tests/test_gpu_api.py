"""The reference's solver / acceptance tests (pkg/tests/test_solver.py,
test_acceptance.py), run against this package's API on the GPU."""

import io
import json

import numpy as np
import pytest

from paper_1901_10084_b200 import core, instances, schedule, solver
from paper_1901_10084_b200.solver import SolverConfig, SolverError

pytestmark = pytest.mark.gpu


@pytest.fixture
def small_instance():
    return instances.random_instance(6, seed=123)


def test_config_validation():
    SolverConfig().validate()
    for bad in (dict(workers=0), dict(tile_size=0), dict(schedule_kind="zigzag"),
                dict(schedule_kind="serial", workers=2), dict(tol_gap=0.0), dict(fixed_passes=0)):
        with pytest.raises(ValueError):
            SolverConfig(**bad).validate()


def test_fixed_passes_step_count(small_instance):
    """test_solver.py:45-53 / acceptance 8: steps = passes * constraint_count."""
    inst = small_instance
    expected = core.constraint_count(inst.n)
    for cfg in (SolverConfig(schedule_kind="serial", fixed_passes=4),
                SolverConfig(workers=3, tile_size=2, fixed_passes=4)):
        sol = solver.solve(inst, cfg)
        assert sol.passes_run == 4 and sol.total_steps == 4 * expected
    sol = solver.solve(instances.random_instance(15, seed=0), SolverConfig(fixed_passes=20))
    assert sol.total_steps == 31500


def test_results_identical_across_worker_counts():
    inst = instances.random_instance(11, seed=3)
    base = solver.solve(inst, SolverConfig(workers=1, tile_size=3, fixed_passes=6))
    for p in (2, 3, 5):
        sol = solver.solve(inst, SolverConfig(workers=p, tile_size=3, fixed_passes=6))
        assert np.array_equal(sol.state.xv, base.state.xv)
        assert np.array_equal(sol.state.fv, base.state.fv)


def test_diagonal_and_tiled_b1_identical():
    inst = instances.random_instance(9, seed=4)
    a = solver.solve(inst, SolverConfig(workers=2, schedule_kind="diagonal", fixed_passes=5))
    b = solver.solve(inst, SolverConfig(workers=2, tile_size=1, fixed_passes=5))
    assert np.array_equal(a.state.xv, b.state.xv)


def test_gap_shrinks_and_stats_consistent(small_instance):
    sol = solver.solve(small_instance, SolverConfig(fixed_passes=300))
    gaps = [s.duality_gap for s in sol.stats]
    assert abs(gaps[-1]) < 1e-6 * max(abs(g) for g in gaps[:10])
    assert sol.stats[-1].max_violation < 1e-8
    for s in sol.stats:
        assert s.duality_gap == pytest.approx(s.primal_objective - s.dual_objective, abs=1e-12)
        assert s.max_violation >= 0 and s.wall_time >= 0


def test_max_violation_reported_matches_state(small_instance):
    sol = solver.solve(small_instance, SolverConfig(max_passes=2000, tol_gap=1e-6,
                                                    tol_violation=1e-6))
    assert sol.converged
    fresh = core.max_violation(small_instance, sol.state)
    assert fresh <= sol.stats[-1].max_violation + 1e-12


def test_stats_stream(small_instance):
    buf = io.StringIO()
    sol = solver.solve(small_instance, SolverConfig(fixed_passes=3), stats_stream=buf)
    lines = buf.getvalue().splitlines()
    assert len(lines) == 3 and json.loads(lines[-1])["pass_index"] == 2
    assert sol.pass_seconds > 0


def test_epsilon_override():
    inst = instances.random_instance(5, seed=8)
    direct = solver.solve(core.ProblemInstance(5, inst.D, inst.Wt, epsilon=0.9),
                          SolverConfig(fixed_passes=5))
    override = solver.solve(inst, SolverConfig(fixed_passes=5, epsilon=0.9))
    assert np.array_equal(direct.state.xv, override.state.xv)
    assert np.array_equal(direct.state.fv, override.state.fv)


def test_nonfinite_state_raises():
    inst = instances.random_instance(5, seed=8)
    plan = solver.Plan(5, SolverConfig())
    state, duals = solver.initialize(inst)
    state.xv[0] = np.nan
    with pytest.raises(SolverError, match="non-finite"):
        solver.run_pass(state, duals, inst, plan)


def test_run_pass_sequence_equals_solve():
    inst = instances.random_instance(13, seed=5)
    cfg = SolverConfig(tile_size=4, fixed_passes=6)
    sol = solver.solve(inst, cfg)
    plan = solver.Plan(inst.n, cfg)
    state, duals = solver.initialize(inst, 2)
    for k in range(6):
        st = solver.run_pass(state, duals, inst, plan, pass_index=k)
        assert st.pass_index == k
    assert np.array_equal(state.xv, sol.state.xv)
    assert np.array_equal(duals.metric_arrays()[0], sol.duals.metric_arrays()[0])
    assert core.dual_objective(inst, duals) == pytest.approx(
        core.dual_objective_from_state(inst, state, duals), rel=1e-10, abs=1e-10)


def test_kkt_report_at_convergence(small_instance):
    """test_solver.py:140-150 / acceptance 7."""
    inst = small_instance
    sol = solver.solve(inst, SolverConfig(workers=2, tile_size=2, max_passes=5000, tol_gap=1e-8,
                                          tol_violation=1e-8))
    assert sol.converged
    report = solver.kkt_report(inst, sol.state, sol.duals)
    assert report["state_relation_residual"] < 1e-10
    assert report["min_stored_dual"] > 0
    assert report["max_violation"] <= 1e-8
    assert report["complementary_slackness"] < 1e-6


def test_unique_optimum_across_schedules():
    """Acceptance 6: every schedule converges to the same optimum."""
    configs = [dict(schedule_kind="serial"), dict(workers=2, tile_size=2),
               dict(workers=4, tile_size=5), dict(workers=8, tile_size=8),
               dict(tile_size=40)]
    for n in (20, 40):
        inst = instances.random_instance(n, seed=n)
        results = []
        for kw in configs:
            sol = solver.solve(inst, SolverConfig(max_passes=5000, tol_gap=1e-6,
                                                  tol_violation=1e-6, **kw))
            assert sol.converged, (n, kw)
            results.append(sol.state.X())
        for other in results[1:]:
            assert np.max(np.abs(other - results[0])) <= 1e-4


def test_worked_example():
    """Acceptance 4 through a one-pass solve on n=3: x_01=1 violates the
    triangle; one step moves to (2/3, 1/3, 1/3) with dual eps/3."""
    eps = 0.7
    inst = core.ProblemInstance(3, np.zeros((3, 3)), np.ones((3, 3)) - np.eye(3), epsilon=eps)
    sess = solver.DeviceSession(inst, "serial", 40)
    xv = np.zeros(3)
    xv[core.pair_index(3, 0, 1)] = 1.0
    fv = np.full(3, 1e6)  # large slack: the pair rows stay inactive
    sess.set_state(xv, fv)
    sess.run(1)
    x, _ = sess.state()
    assert abs(x[core.pair_index(3, 0, 1)] - 2 / 3) <= 1e-15
    assert abs(x[core.pair_index(3, 0, 2)] - 1 / 3) <= 1e-15
    keys, vals, _ = sess.duals()
    assert len(keys) == 1 and abs(vals[0] - eps / 3) <= 1e-15


def test_accumulate_aty_bitwise_reference_golden():
    """mp_accumulate_aty = core.accumulate_aty (core.py:285-293) bit for bit on
    the reference's own outputs (tests/golden/aty.npz: a random two-worker
    store and the reference's duals after 6 passes of config 1), and
    dual_objective (core.py:320-327) on top of it."""
    import os
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "aty.npz"))
    for p in ("r", "c"):
        n = int(z[p + "_n"])
        inst = instances.random_instance(n, seed=7) if p == "r" else instances.config_instance(1)
        assert np.array_equal(inst.c_vector(), z[p + "_c"])
        d = core.DualStore(n, 1)
        d.keys, d.vals = [z[p + "_keys"]], [z[p + "_vals"]]
        d.pair_duals = z[p + "_pd"].copy()
        assert np.array_equal(core.accumulate_aty(inst, d), z[p + "_g"]), p
        assert core.dual_objective(inst, d) == pytest.approx(float(z[p + "_dual"]), rel=1e-13)


def test_accumulate_aty_config2_duals_bitwise_oracle():
    """At config-2 size (n = 1000, the GPU session's own duals after 8 passes)
    the device accumulation equals the oracle's reference-order one."""
    from oracle import oracle
    inst = instances.config_instance(2)
    sol = solver.solve(inst, SolverConfig(fixed_passes=8))
    k, v = sol.duals.metric_arrays()
    assert len(k) > 10000
    g = core.accumulate_aty(inst, sol.duals)
    ref = oracle.accumulate_aty_np(inst.n, k, v, sol.duals.pair_duals, inst.c_vector())
    assert np.array_equal(g, ref)
    # Dykstra invariant c + A'y = -eps W v (solver.py:256-281)
    target = -inst.epsilon * np.concatenate([inst.reg_x * sol.state.xv, inst.reg_f * sol.state.fv])
    assert np.max(np.abs(g - target)) <= 1e-9 * max(1.0, np.max(np.abs(target)))


def test_accumulate_aty_edge_cases():
    inst = instances.random_instance(5, seed=1)
    d = core.DualStore(5, 1)                      # empty store: g = c exactly
    assert np.array_equal(core.accumulate_aty(inst, d), inst.c_vector())
    d.keys, d.vals = [np.array([((3 * 5 + 1) * 5 + 2) * 3], dtype=np.int64)], [np.array([1.0])]
    from paper_1901_10084_b200 import _native
    with pytest.raises(_native.NativeError) as ei:  # i > j: not a metric key
        core.accumulate_aty(inst, d)
    assert ei.value.code == _native.MP_ERR_ARG


def test_dykstra_step_bitwise_reference_golden():
    """projection.dykstra_step (projection.py:63-87) on the device through
    mp_dykstra_steps: the reference's own single-row steps (tests/golden/
    steps.npz: all five kinds, general W, y_old = 0 and > 0, applied in
    sequence) bit for bit, plus the worked example and the y_old < 0 error."""
    import paper_1901_10084_b200 as mp
    from conftest import golden
    g = golden("steps")
    for c in range(6):
        n, eps = int(g[f"c{c}_n"]), float(g[f"c{c}_eps"])
        m = n * (n - 1) // 2
        inst = core.ProblemInstance(n, g[f"c{c}_D"], np.ones((n, n)) - np.eye(n), epsilon=eps,
                                    reg_x=g[f"c{c}_regx"].copy(), reg_f=g[f"c{c}_regf"].copy())
        st = core.PrimalState(n, g[f"c{c}_x0"].copy(), g[f"c{c}_f0"].copy())
        for t, (kind, i, j, k) in enumerate(g[f"c{c}_keys"]):
            key = core.ConstraintKey(core.Kind(int(kind)), int(i), int(j), int(k))
            o = mp.dykstra_step(st, key, float(g[f"c{c}_y"][t]), inst)
            assert isinstance(o, mp.StepOutcome)
            assert o.theta_plus == g[f"c{c}_theta"][t] and o.changed == bool(g[f"c{c}_changed"][t])
        assert np.array_equal(st.xv, g[f"c{c}_x1"]) and np.array_equal(st.fv, g[f"c{c}_f1"]), c
        assert len(st.xv) == m
    # worked example (reference tests/test_acceptance.py:86-98)
    inst3 = core.ProblemInstance(3, np.zeros((3, 3)), np.ones((3, 3)) - np.eye(3), epsilon=0.7)
    st3 = core.PrimalState(3)
    st3.set_x(0, 1, 1.0)
    o = mp.dykstra_step(st3, core.ConstraintKey(core.Kind.METRIC_IJ, 0, 1, 2), 0.0, inst3)
    sg = golden("small_cases")
    assert np.array_equal(st3.xv, sg["worked_x"]) and o.theta_plus == float(sg["worked_theta"])
    with pytest.raises(ValueError):
        mp.dykstra_step(st3, core.ConstraintKey(core.Kind.METRIC_IJ, 0, 1, 2), -1.0, inst3)


def test_workers_give_the_reference_per_worker_dual_layout():
    """solve / run_pass with workers = 8: DualStore.keys[w] / vals[w] are the
    reference's per-worker arrays (core.py:218-236) -- the golden hashes of
    config 2 were taken over np.concatenate(duals.keys) of the unmodified
    reference run with 8 workers."""
    import hashlib
    from conftest import golden
    from paper_1901_10084_b200 import solver as S

    def sha(a):
        return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
    g = golden("config2_n1000_b40_p4")
    inst = instances.config_instance(2)
    cfg = S.SolverConfig(workers=8, tile_size=40, schedule_kind="tiled", fixed_passes=int(g["passes"]))
    plan = S.Plan(inst.n, cfg)
    state, duals = S.initialize(inst, 8)
    for k in range(int(g["passes"])):
        S.run_pass(state, duals, inst, plan, pass_index=k)
        assert len(duals.keys) == 8
        keys = np.concatenate(duals.keys) if duals.nnz() else np.empty(0, np.int64)
        vals = np.concatenate(duals.vals) if duals.nnz() else np.empty(0)
        assert sha(keys) == g["dkeys_sha"][k] and sha(vals) == g["dvals_sha"][k], k
        assert sha(state.xv) == g["xsha"][k]
    sol = S.solve(inst, cfg)
    assert sha(np.concatenate(sol.duals.keys)) == g["dkeys_sha"][-1]
    assert sha(np.concatenate(sol.duals.vals)) == g["dvals_sha"][-1]
    assert sum(len(k_) > 0 for k_ in sol.duals.keys) > 1
