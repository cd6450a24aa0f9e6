"""Parity at the BASELINE configs' full sizes.

Config 3 (n = 4000) is small enough for the CPU oracle to replay a few
passes on all host threads, so it is checked bit for bit.  Configs 4 and 5
(n = 10000 / 18000, 5e11 / 2.9e12 rows per pass) are not: there the checks
are size-independent properties of the reference's algorithm --

* sharding: the tiles of a round are conflict-free (schedule.py:235-250), so
  splitting them over ranks (LocalShardGroup: per-rank launch shapes, the
  footprint exchange) must follow the single-session trajectory bit for bit;
* resumability: x, f and the duals are the whole solver state (core.py:218-256),
  so exporting them and importing into a fresh session must continue the run
  bit for bit (the reference's own resume path, solver.py:264-275);
* the exported duals are valid reference keys (core.py:81-94) with theta > 0,
  and their count is the pass's nnz_metric.

Config 5's biggest rounds hold more tiles than the GPU co-schedules, so they
run as 2-CTA clusters in waves, which no smaller config reaches.
"""

import os

import numpy as np
import pytest

from paper_1901_10084_b200 import distributed, instances
from paper_1901_10084_b200.solver import DeviceSession

pytestmark = pytest.mark.gpu

B = 40


def _valid_keys(keys, vals, n):
    kind = keys % 3
    t = keys // 3
    k = t % n
    t //= n
    j = t % n
    i = t // n
    assert np.all((0 <= i) & (i < j) & (j < k) & (k < n))
    assert np.all((kind >= 0) & (kind <= 2))
    assert np.all(vals > 0.0) and np.all(np.isfinite(vals))


def test_config3_full_size_bitwise_oracle(oracle_lib):
    inst = instances.config_instance(3)  # n = 4000 Chung-Lu, gamma = 10, lambda = 0.5
    sess = DeviceSession(inst, "tiled", B)
    ref = oracle_lib.OracleSolver(inst.n, inst.d_flat, inst.w_flat, inst.epsilon, b=B,
                                  workers=os.cpu_count() or 1)
    for k in range(3):
        st = sess.run(1)[0]
        rs = ref.run_pass()
        assert st.max_violation == rs.max_violation, k
        assert st.primal_objective == pytest.approx(rs.primal_objective, rel=1e-12)
        x, f = sess.state()
        rx, rf = ref.state()
        assert np.array_equal(x, rx) and np.array_equal(f, rf), k
    keys, vals, pd = sess.duals()
    rk, rv = ref.duals()
    assert len(keys) == st.nnz_metric > 0
    o1, o2 = np.argsort(keys), np.argsort(rk)
    assert np.array_equal(keys[o1], rk[o2]) and np.array_equal(vals[o1], rv[o2])
    assert np.array_equal(pd, ref.pair_duals())
    ref.close()
    sess.close()


def _sharded_and_resumed(config, passes, world):
    inst = instances.config_instance(config)
    single = DeviceSession(inst, "tiled", B)
    grp = distributed.LocalShardGroup(inst, world, B)
    for k in range(passes):
        a = single.run(1)[0]
        g = grp.run(1)[0]
        assert (a.nnz_metric, a.max_violation, a.primal_objective) == \
               (g.nnz_metric, g.max_violation, g.primal_objective), k
    x, f = single.state()
    for r in range(world):
        gx, gf = grp.state(r)
        assert np.array_equal(gx, x) and np.array_equal(gf, f), r
    keys, vals, pd = single.duals()
    gk, gv = grp.duals()
    assert np.array_equal(gk, keys) and np.array_equal(gv, vals)
    assert len(keys) == a.nnz_metric > 0
    _valid_keys(keys, vals, inst.n)
    grp.close()

    # export -> import into a fresh session -> one more pass on both
    fresh = DeviceSession(inst, "tiled", B)
    fresh.set_state(x, f)
    fresh.set_duals(keys, vals, pd)
    a = single.run(1)[0]
    c = fresh.run(1)[0]
    assert (a.nnz_metric, a.max_violation) == (c.nnz_metric, c.max_violation)
    x1, f1 = single.state()
    x2, f2 = fresh.state()
    assert np.array_equal(x1, x2) and np.array_equal(f1, f2)
    fresh.close()
    single.close()


def test_config4_full_size_sharded_and_resumed():
    # n = 10000 planted partition (the BASELINE's sharded config), 2 ranks
    _sharded_and_resumed(4, passes=2, world=2)


def test_config5_full_size_sharded_and_resumed():
    # n = 18000 Chung-Lu: the biggest rounds run 2-CTA clusters in waves
    _sharded_and_resumed(5, passes=2, world=2)


def test_one_cta_tiles_long_rings_deterministic(knobs):
    """One CTA per tile (MP_CLUSTER=1) at n = 7000: every tile's j-rings wrap
    ~27 times, so a WK slot written back element by element is refilled by a
    TMA box many times per pass.  Regression for a missing producer barrier
    between the two (it showed as run-to-run differences at n >= 7000 only):
    repeated runs and the element-copy staging must agree bit for bit -- and
    so must clusters run in waves (MP_FORCE_C: 8-CTA clusters for every
    round, 88 tiles x 8 CTAs in the biggest rounds) and the default plan."""
    import hashlib
    inst = instances.config_instance(4, n=7000)
    hashes = set()
    for env in [{"MP_CLUSTER": "1"}, {"MP_CLUSTER": "1"}, {"MP_CLUSTER": "1", "MP_NO_TMA": "1"},
                {"MP_FORCE_C": "8"}, {}]:
        for k in ("MP_CLUSTER", "MP_NO_TMA", "MP_FORCE_C"):
            knobs.delenv(k, raising=False)
        for k, v in env.items():
            knobs.setenv(k, v)
        s = DeviceSession(inst, "tiled", B)
        s.run(2)
        x, f = s.state()
        hashes.add(hashlib.sha1(x.tobytes() + f.tobytes()).hexdigest())
        s.close()
    assert len(hashes) == 1


@pytest.mark.parametrize("env", [{"MP_FORCE_C": "8"}, {"MP_FORCE_C": "2"}, {"MP_FORCE_C": "2", "MP_U": "8"},
                                 {"MP_DF_C": "2", "MP_U": "8"}, {}])
def test_cluster_waves_bitwise_oracle(oracle_lib, knobs, env):
    """Clusters in waves (more tiles in a round than the device co-schedules
    as clusters: n = 1400 has rounds of 17 tiles, 8-CTA clusters fit 15 at a
    time) against the oracle, bit for bit, on a Chung-Lu instance (hub rows).
    The 2-CTA shape runs batches of 4 levels (its chain of warps does not fit
    the W = 256 ring with 8, round_shape) -- and batches of 8 with MP_U=8."""
    for k, v in env.items():
        knobs.setenv(k, v)
    inst = instances.config_instance(3, n=1400)
    sess = DeviceSession(inst, "tiled", B)
    ref = oracle_lib.OracleSolver(inst.n, inst.d_flat, inst.w_flat, inst.epsilon, b=B,
                                  workers=os.cpu_count() or 1)
    for _ in range(4):
        st = sess.run(1)[0]
        rs = ref.run_pass()
        assert st.max_violation == rs.max_violation
    x, f = sess.state()
    rx, rf = ref.state()
    assert np.array_equal(x, rx) and np.array_equal(f, rf)
    keys, vals, _ = sess.duals()
    rk, rv = ref.duals()
    assert len(keys) > 0
    o1, o2 = np.argsort(keys), np.argsort(rk)
    assert np.array_equal(keys[o1], rk[o2]) and np.array_equal(vals[o1], rv[o2])
    ref.close()
    sess.close()
