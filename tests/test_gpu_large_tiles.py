"""Tile sizes above one CTA's capacity (b > 48, schedule.py:117-153 accepts
any tile_size >= 1, solver.py:42-43; the paper sweeps b up to 50):
every round runs as clusters (the smallest cluster that holds a tile when a
round has more tiles than fit), bitwise equal to the CPU oracle, with the
dataflow launch and a dual export -> import resume.  The device limit: the
ring must hold a warp's j-window of 2b - 2 (b <= 64 with W = I, b <= 48 with
general W); beyond it mp_create refuses the tile size."""

import numpy as np
import pytest

from paper_1901_10084_b200 import instances
from paper_1901_10084_b200.solver import DeviceSession

pytestmark = pytest.mark.gpu


def compare(sess, ref, passes):
    for _ in range(passes):
        st = sess.run(1)[0]
        rs = ref.run_pass()
        assert st.max_violation == rs.max_violation
        assert st.steps == rs.steps
    x, f = sess.state()
    rx, rf = ref.state()
    assert np.array_equal(x, rx) and np.array_equal(f, rf)
    keys, vals, pd = sess.duals()
    rk, rv = ref.duals()
    o1, o2 = np.argsort(keys), np.argsort(rk)
    assert np.array_equal(keys[o1], rk[o2]) and np.array_equal(vals[o1], rv[o2])
    assert np.array_equal(pd, ref.pair_duals())


@pytest.mark.parametrize("config,n,b,passes", [(3, 420, 50, 4), (2, 500, 64, 4), (1, 300, 64, 6),
                                               (3, 640, 56, 3), (4, 520, 64, 3), (5, 611, 64, 3)])
def test_large_tiles_against_oracle(oracle_lib, config, n, b, passes):
    inst = instances.config_instance(config, n=n)
    sess = DeviceSession(inst, "tiled", b)
    ref = oracle_lib.OracleSolver(inst.n, inst.d_flat, inst.w_flat, inst.epsilon, b=b, workers=4)
    compare(sess, ref, passes)
    sess.close()
    ref.close()


@pytest.mark.parametrize("env", [{"MP_NO_DF": "1"}, {"MP_DF_C": "8"}, {"MP_FORCE_C": "4", "MP_NO_DF": "1"},
                                 {"MP_NO_TMA": "1"}])
def test_large_tiles_launch_variants(oracle_lib, knobs, env):
    for k, v in env.items():
        knobs.setenv(k, v)
    inst = instances.config_instance(2, n=390)
    sess = DeviceSession(inst, "tiled", 64)
    ref = oracle_lib.OracleSolver(inst.n, inst.d_flat, inst.w_flat, inst.epsilon, b=64, workers=4)
    compare(sess, ref, 4)
    sess.close()
    ref.close()


@pytest.mark.parametrize("b,general_w", [(96, False), (64, True)])
def test_tiles_beyond_the_ring_are_refused(b, general_w):
    """A tile whose j-window (2b - 2) does not fit the shared-memory ring of
    any launch shape (b = 96 with W = I; b > 48 with general W, whose ring is
    half as wide) is refused with MP_ERR_UNSUPPORTED instead of running into a
    ring deadlock."""
    inst = instances.config_instance(1, n=300)
    if general_w:
        rng = np.random.default_rng(3)
        inst.reg_x = rng.uniform(0.5, 2.0, inst.npairs)
        inst.reg_f = rng.uniform(0.5, 2.0, inst.npairs)
    with pytest.raises(NotImplementedError, match="does not fit"):  # MP_ERR_UNSUPPORTED
        DeviceSession(inst, "tiled", b)


def test_large_tiles_dual_import_resume(oracle_lib):
    inst = instances.config_instance(3, n=450)
    a = DeviceSession(inst, "tiled", 64)
    a.run(3)
    x, f = a.state()
    keys, vals, pd = a.duals()
    b_ = DeviceSession(inst, "tiled", 64)
    b_.set_state(x, f)
    b_.set_duals(keys, vals, pd)
    sa = a.run(2)
    sb = b_.run(2)
    assert [s.max_violation for s in sa] == [s.max_violation for s in sb]
    xa, fa = a.state()
    xb, fb = b_.state()
    assert np.array_equal(xa, xb) and np.array_equal(fa, fb)
