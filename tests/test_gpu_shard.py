"""Sharded execution of one instance on the device: every
rank of a LocalShardGroup runs through the same per-round code as an NCCL
rank (own tiles, pack of the footprint blocks for their next touchers' ranks,
exchange, unpack, counter all-reduce), so the group must follow the
single-session trajectory bit for bit -- on every rank, although between the
pair phases a rank's x is current only where it is about to be read."""

import numpy as np
import pytest

from oracle import oracle
from paper_1901_10084_b200 import distributed, instances
from paper_1901_10084_b200.solver import DeviceSession

pytestmark = pytest.mark.gpu


def _same_stats(a, b):
    for sa, sb in zip(a, b):
        assert sa.nnz_metric == sb.nnz_metric
        assert sa.max_violation == sb.max_violation
        assert sa.primal_objective == sb.primal_objective
        assert sa.dual_objective == sb.dual_objective


@pytest.mark.parametrize("world", [2, 3, 4])
def test_local_group_equals_single_session(world):
    inst = instances.config_instance(1)  # n = 100, b = 40
    ref = DeviceSession(inst, "tiled", 40)
    grp = distributed.LocalShardGroup(inst, world, 40)
    for _ in range(3):
        _same_stats(grp.run(1), ref.run(1))
    x, f = ref.state()
    for g in range(world):
        gx, gf = grp.state(g)
        assert np.array_equal(gx, x) and np.array_equal(gf, f)
    keys, vals, _ = ref.duals()
    gk, gv = grp.duals()
    assert np.array_equal(gk, keys) and np.array_equal(gv, vals)
    assert sum(s.dual_count() for s in grp.members) == len(keys)
    grp.close()
    ref.close()


@pytest.mark.parametrize("n,b,world,general_w", [(300, 16, 4, False), (240, 12, 3, True),
                                                 (500, 40, 2, False)])
def test_local_group_matches_oracle(n, b, world, general_w):
    inst = instances.config_instance(2, n=n) if not general_w else instances.config_instance(1, n=n)
    rx = rf = None
    if general_w:
        rng = np.random.default_rng(n)
        rx = rng.uniform(0.5, 2.0, inst.npairs)
        rf = rng.uniform(0.5, 2.0, inst.npairs)
        inst.reg_x, inst.reg_f = rx, rf
    grp = distributed.LocalShardGroup(inst, world, b)
    ref = oracle.OracleSolver(n, inst.d_flat, inst.w_flat, inst.epsilon, reg_x=rx, reg_f=rf,
                              b=b, workers=4)
    for _ in range(3):
        st = grp.run(1)[0]
        rs = ref.run_pass()
        assert st.max_violation == rs.max_violation
    x, f = grp.state(world - 1)
    rx, rf = ref.state()
    assert np.array_equal(x, rx) and np.array_equal(f, rf)
    gk, gv = grp.duals()
    rk, rv = ref.duals()
    assert np.array_equal(np.sort(gk), np.sort(rk))
    grp.close()


def test_exchange_volume_follows_the_route_plan():
    """Each member packs what the host plan routes from it (rectangles: the
    pairs plus padding at the diagonal), what is sent is received, and the
    plan moves far less than an all-gather of every footprint."""
    from paper_1901_10084_b200 import schedule
    n, b, world = 300, 16, 4
    inst = instances.config_instance(2, n=n)
    grp = distributed.LocalShardGroup(inst, world, b)
    vol = distributed.native_route_volumes(n, b, world)
    sent = recv = 0
    for g, s in enumerate(grp.members):
        sv, rv = s.exchange_volume()
        assert vol[:, g, :].sum() <= sv <= 1.5 * vol[:, g, :].sum()
        assert vol[:, :, g].sum() <= rv <= 1.5 * vol[:, :, g].sum()
        sent += sv
        recv += rv
    assert sent == recv
    assert sent < 0.5 * (world - 1) * schedule.touched_pairs(n, b)
    grp.close()
    s = DeviceSession(inst, "tiled", b)
    assert s.exchange_volume() == (0, 0)
    s.close()


def test_local_group_resumes_from_imported_duals():
    inst = instances.random_instance(150, seed=7)
    ref = oracle.OracleSolver(inst.n, inst.d_flat, inst.w_flat, inst.epsilon, b=20, workers=4)
    for _ in range(2):
        ref.run_pass()
    rx, rf = ref.state()
    rk, rv = ref.duals()
    grp = distributed.LocalShardGroup(inst, 3, 20)
    for s in grp.members:
        s.set_state(rx, rf)
    grp.set_duals(rk, rv, ref.pair_duals())
    assert sum(s.dual_count() for s in grp.members) == len(rk)
    grp.run(2)
    ref.run_pass()
    ref.run_pass()
    x, f = grp.state(1)
    ex, ef = ref.state()
    assert np.array_equal(x, ex) and np.array_equal(f, ef)
    grp.close()


def test_nccl_one_rank_communicator():
    """The NCCL set-up path (unique id, dlopen'd NCCL, communicator) on one
    GPU; with one rank the pass has no exchange and equals an unsharded one."""
    from paper_1901_10084_b200 import _native
    import ctypes
    inst = instances.config_instance(1)
    buf = ctypes.create_string_buffer(128)
    _native.check(_native.load().mp_nccl_unique_id(buf), "mp_nccl_unique_id")
    s = DeviceSession(inst, "tiled", 40)
    s.shard(1, 0, buf.raw)
    ref = DeviceSession(inst, "tiled", 40)
    _same_stats(s.run(2), ref.run(2))
    assert np.array_equal(s.state()[0], ref.state()[0])
    s.close()
    ref.close()


def test_shard_rejects_bad_use():
    inst = instances.config_instance(1)
    s = DeviceSession(inst, "tiled", 40)
    s.run(1)
    with pytest.raises(ValueError):
        s.shard(2, 0)  # after the first pass
    s.close()
    s = DeviceSession(inst, "serial", 40)
    with pytest.raises(NotImplementedError):
        s.shard(2, 0)
    s.close()
    s = DeviceSession(inst, "tiled", 40)
    s.shard(2, 1)
    with pytest.raises(Exception):
        s.run(1)  # a local shard runs only inside its group
    s.close()
