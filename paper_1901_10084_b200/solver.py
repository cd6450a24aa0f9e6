"""Dykstra passes on the GPU behind the reference solver API.

Same public surface as the reference's ``solver.py`` (``SolverConfig``,
``Solution``, ``SolverError``, ``Plan``, ``initialize``, ``run_pass``,
``solve``, ``kkt_report``), but every pass runs inside the native library:
``solve`` opens one :class:`DeviceSession` (``mp_create``), keeps x, f and all
duals resident in HBM, and calls ``mp_run_passes`` once per pass, pulling
back only the ~64-byte ``PassStats`` (and x, f, duals once at the end).

``workers`` is accepted and validated for compatibility; on the device the
schedule alone fixes the trajectory (the reference's results are identical
for every worker count, reference tests/test_solver.py:56-66).
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native, core, schedule
from .core import DualStore, PassStats, PrimalState, ProblemInstance

SCHEDULE_KINDS = ("serial", "diagonal", "tiled")


class SolverError(RuntimeError):
    """Non-finite state after a pass (solver.py:24-25, :200-201)."""


@dataclass
class SolverConfig:
    """solver.py:28-51, plus the CUDA device ordinal."""
    workers: int = 1
    tile_size: int = 40
    epsilon: Optional[float] = None
    max_passes: int = 100
    fixed_passes: Optional[int] = None
    tol_gap: float = 1e-4
    tol_violation: float = 1e-4
    schedule_kind: str = "tiled"
    device: int = 0

    def validate(self):
        if self.workers < 1:
            raise ValueError(f"workers must be >= 1, got {self.workers}")
        if self.tile_size < 1:
            raise ValueError(f"tile_size must be >= 1, got {self.tile_size}")
        if self.schedule_kind not in SCHEDULE_KINDS:
            raise ValueError(f"unknown schedule_kind {self.schedule_kind!r}")
        if self.schedule_kind == "serial" and self.workers != 1:
            raise ValueError("serial schedule requires workers = 1")
        if self.tol_gap <= 0 or self.tol_violation <= 0:
            raise ValueError("tolerances must be positive")
        if self.fixed_passes is not None and self.fixed_passes < 1:
            raise ValueError("fixed_passes must be >= 1")


@dataclass
class Solution:
    state: PrimalState
    stats: list
    converged: bool
    passes_run: int
    total_steps: int = 0
    duals: DualStore = None

    @property
    def pass_seconds(self):
        """Device time of the pass loop (the benchmark quantity, solver.py:63-66)."""
        return sum(s.wall_time for s in self.stats)


class DeviceSession:
    """One ``mp_handle``: instance, state and duals resident on one GPU."""

    def __init__(self, instance: ProblemInstance, schedule_kind="tiled", tile_size=40,
                 device=0, time_rounds=True):
        L = _native.load()
        self.n = instance.n
        self.m = instance.npairs
        self._keep = [np.ascontiguousarray(instance.d_flat, dtype=np.float64),
                      np.ascontiguousarray(instance.w_flat, dtype=np.float64),
                      np.ascontiguousarray(instance.reg_x, dtype=np.float64),
                      np.ascontiguousarray(instance.reg_f, dtype=np.float64)]
        inst = _native.MPInstance(self.n, *(_native.dptr(a) for a in self._keep),
                                  instance.epsilon)
        cfg = _native.MPConfig(_native.SCHEDULE_CODES[schedule_kind], int(tile_size), int(device),
                               _native.MP_FLAG_TIME_ROUNDS if time_rounds else 0)
        h = ctypes.c_void_p()
        rc = L.mp_create(ctypes.byref(inst), ctypes.byref(cfg), ctypes.byref(h))
        if rc == _native.MP_ERR_ARG:
            raise ValueError(_native.last_error())
        if rc == _native.MP_ERR_UNSUPPORTED:
            raise NotImplementedError(_native.last_error())
        _native.check(rc, "mp_create")
        self._h = h
        self._keep = None
        self.version = 0  # bumps on every pass / state change

    def close(self):
        if getattr(self, "_h", None):
            _native.load().mp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self, npasses=1):
        """Run npasses passes; returns the list of MPPassStats.  Raises
        SolverError on a non-finite state (stats of that pass are attached)."""
        out = (_native.MPPassStats * max(npasses, 1))()
        rc = _native.load().mp_run_passes(self._h, npasses, out)
        self.version += 1
        if rc == _native.MP_ERR_NONFINITE:
            err = SolverError(_native.last_error())
            err.stats = list(out)
            raise err
        _native.check(rc, "mp_run_passes")
        return list(out)[:npasses]

    def state(self):
        x = np.empty(self.m)
        f = np.empty(self.m)
        _native.check(_native.load().mp_get_state(self._h, _native.dptr(x), _native.dptr(f)),
                      "mp_get_state")
        return x, f

    def set_state(self, x, f):
        x = np.ascontiguousarray(x, dtype=np.float64)
        f = np.ascontiguousarray(f, dtype=np.float64)
        _native.check(_native.load().mp_set_state(self._h, _native.dptr(x), _native.dptr(f)),
                      "mp_set_state")
        self.version += 1

    def dual_count(self):
        return int(_native.load().mp_dual_count(self._h))

    def duals(self):
        """(keys, vals, pair_duals) with keys in single-worker visit order."""
        c = self.dual_count()
        keys = np.empty(c, dtype=np.int64)
        vals = np.empty(c)
        pd = np.empty((self.m, 2))
        _native.check(_native.load().mp_get_duals(self._h, _native.iptr(keys), _native.dptr(vals),
                                                  _native.dptr(pd)), "mp_get_duals")
        return keys, vals, pd

    def set_duals(self, keys, vals, pair_duals=None):
        keys = np.ascontiguousarray(keys, dtype=np.int64)
        vals = np.ascontiguousarray(vals, dtype=np.float64)
        pd = None if pair_duals is None else np.ascontiguousarray(pair_duals, dtype=np.float64)
        rc = _native.load().mp_set_duals(self._h, len(keys), _native.iptr(keys),
                                         _native.dptr(vals),
                                         _native.dptr(pd) if pd is not None else None)
        if rc == _native.MP_ERR_ARG:
            raise ValueError(_native.last_error())
        _native.check(rc, "mp_set_duals")
        self.version += 1

    def shard(self, world, rank, nccl_id=None):
        """Make this fresh session rank ``rank`` of ``world`` (mp_shard): with
        a 128-byte NCCL id the ranks are processes, without one the session is
        a member of a distributed.LocalShardGroup."""
        rc = _native.load().mp_shard(self._h, int(world), int(rank),
                                     None if nccl_id is None else bytes(nccl_id))
        if rc == _native.MP_ERR_ARG:
            raise ValueError(_native.last_error())
        if rc == _native.MP_ERR_UNSUPPORTED:
            raise NotImplementedError(_native.last_error())
        _native.check(rc, "mp_shard")

    def exchange_volume(self):
        """(sent, received): 8-byte values this rank moves per pass under the
        next-toucher exchange plan (mp_shard_volume; 0, 0 when unsharded)."""
        import ctypes
        a, b = ctypes.c_int64(), ctypes.c_int64()
        _native.check(_native.load().mp_shard_volume(self._h, ctypes.byref(a), ctypes.byref(b)),
                      "mp_shard_volume")
        return a.value, b.value

    def duals_ranked(self):
        """(keys, vals, order): this session's metric duals in visit order and
        the schedule index of each entry's tile (mp_get_duals_ranked)."""
        c = self.dual_count()
        keys = np.empty(c, dtype=np.int64)
        vals = np.empty(c)
        order = np.empty(c, dtype=np.int64)
        _native.check(_native.load().mp_get_duals_ranked(self._h, _native.iptr(keys),
                                                         _native.dptr(vals), _native.iptr(order)),
                      "mp_get_duals_ranked")
        return keys, vals, order

    def max_violation(self):
        out = np.zeros(1)
        _native.check(_native.load().mp_state_max_violation(self._h, _native.dptr(out)),
                      "mp_state_max_violation")
        return float(out[0])

    def timing(self):
        """(metric-phase ms, pair-phase ms, kernel launches) of the last run()."""
        a = np.zeros(1)
        b = np.zeros(1)
        c = np.zeros(1, dtype=np.int64)
        _native.check(_native.load().mp_get_timing(self._h, _native.dptr(a), _native.dptr(b),
                                                   _native.iptr(c)), "mp_get_timing")
        return float(a[0]), float(b[0]), int(c[0])

    def flush_l2(self):
        _native.check(_native.load().mp_flush_l2(self._h), "mp_flush_l2")


class Plan:
    """Schedule of one solve (solver.py:69-105).  ``rounds`` is the host
    mirror of the schedule the device runs; the device session is created
    lazily on first ``run_pass``."""

    def __init__(self, n, config):
        config.validate()
        self.n = n
        self.config = config
        self.p = config.workers
        self.kind = config.schedule_kind
        self.b = 1 if self.kind == "diagonal" else config.tile_size
        m = core.pair_count(n)
        bounds = [w * m // self.p for w in range(self.p + 1)]
        self.pair_ranges = [(bounds[w], bounds[w + 1]) for w in range(self.p)]
        self._rounds = None
        self._session = None
        self._instance = None

    @property
    def rounds(self):
        if self.kind == "serial":
            return None
        if self._rounds is None:
            self._rounds = (schedule.diagonal_rounds(self.n) if self.kind == "diagonal"
                            else schedule.tiled_rounds(self.n, self.b))
        return self._rounds

    def session(self, instance):
        if self._session is None or self._instance is not instance:
            if self._session is not None:
                self._session.close()
            self._session = DeviceSession(instance, self.kind, self.b, self.config.device)
            self._instance = instance
        return self._session


def initialize(instance, workers=1):
    """x = 0, f = -w/(eps reg_f), y = 0 (solver.py:108-113)."""
    state = PrimalState(instance.n)
    state.fv[:] = -instance.w_flat / (instance.epsilon * instance.reg_f)
    return state, DualStore(instance.n, workers)


def _to_stats(s, pass_index):
    return PassStats(pass_index=pass_index, primal_objective=s.primal_objective,
                     dual_objective=s.dual_objective, duality_gap=s.duality_gap,
                     max_violation=s.max_violation, wall_time=s.wall_time, steps=s.steps)


def worker_of_keys(keys, n, b, p):
    """Worker that owns each metric dual in a ``workers = p`` reference run:
    triplet (i, j, k) lies in the tile of row block I = ceil(i / b) and column
    block K = (n-1-k) // b, which sits at position I (first family, K >= I) or
    K (second family) of its round and goes to worker (position + 1) mod p
    (schedule.py:79-80, solver.py:86-91).  ``b = 1`` is the diagonal schedule."""
    i, _, k, _ = core.decode_keys(keys, n)
    I = (i + b - 1) // b
    K = (n - 1 - k) // b
    return (np.where(K >= I, I, K) + 1) % p


def _fill_duals(duals, keys, vals, pd, session, b=None, workers=1):
    """Device duals (single-worker visit order) into the store.  With several
    workers the store gets the reference's per-worker layout (core.py:218-236):
    a worker's entries are those of its tiles, in visit order -- a stable
    partition of the single-worker order, since rounds and positions ascend in
    both."""
    p = min(workers, duals.nworkers)  # the plan's workers fill the store (solver.py:192-198)
    rest = duals.nworkers - max(p, 1)
    if p > 1 and b is not None and len(keys):
        w = worker_of_keys(keys, duals.n, b, p)
        duals.keys = [keys[w == q] for q in range(p)]
        duals.vals = [vals[w == q] for q in range(p)]
    else:
        duals.keys, duals.vals, rest = [keys], [vals], duals.nworkers - 1
    duals.keys += [np.empty(0, dtype=np.int64) for _ in range(rest)]
    duals.vals += [np.empty(0) for _ in range(rest)]
    duals.pair_duals = pd
    duals._session = session
    duals._version = session.version


def run_pass(state, duals, instance, plan, pool=None, pass_index=0):
    """One full pass on the given host state (solver.py:166-210): upload,
    run on the device, download into ``state`` / ``duals`` in place."""
    sess = plan.session(instance)
    sess.set_state(state.xv, state.fv)
    if duals._session is not sess or duals._version != sess.version - 1:
        keys, vals = duals.metric_arrays()
        sess.set_duals(keys, vals, duals.pair_duals)
    try:
        st = sess.run(1)[0]
        err = None
    except SolverError as e:
        st, err = e.stats[0], e
    x, f = sess.state()
    state.xv[:] = x
    state.fv[:] = f
    keys, vals, pd = sess.duals()
    _fill_duals(duals, keys, vals, pd, sess, None if plan.kind == "serial" else plan.b, plan.p)
    if err is not None:
        raise SolverError(f"non-finite value in state after pass {pass_index}")
    return _to_stats(st, pass_index)


def _is_converged(stats, config):
    rel_gap = stats.duality_gap / max(1.0, abs(stats.dual_objective))
    return rel_gap <= config.tol_gap and stats.max_violation <= config.tol_violation


def solve(instance, config=None, stats_stream=None):
    """Passes until converged or out of budget; exactly ``fixed_passes``
    passes in benchmark mode (solver.py:218-253)."""
    if config is None:
        config = SolverConfig()
    config.validate()
    if config.epsilon is not None and config.epsilon != instance.epsilon:
        instance = ProblemInstance.from_flat(instance.n, instance.d_flat, instance.w_flat,
                                             epsilon=config.epsilon, reg_x=instance.reg_x,
                                             reg_f=instance.reg_f)
    plan = Plan(instance.n, config)
    sess = plan.session(instance)
    budget = config.fixed_passes if config.fixed_passes is not None else config.max_passes
    stats, total, converged = [], 0, False
    try:
        if config.fixed_passes is not None and stats_stream is None:
            # benchmark mode: every pass in one native call (no host round trip
            # per pass); the native loop stops at the first non-finite pass
            try:
                raws = sess.run(budget)
            except SolverError as e:
                raise SolverError(str(e)) from None
        for k in range(budget):
            if config.fixed_passes is not None and stats_stream is None:
                raw = raws[k]
            else:
                try:
                    raw = sess.run(1)[0]
                except SolverError:
                    raise SolverError(f"non-finite value in state after pass {k}") from None
            st = _to_stats(raw, k)
            stats.append(st)
            total += st.steps
            if stats_stream is not None:
                stats_stream.write(st.to_json() + "\n")
            if config.fixed_passes is None and _is_converged(st, config):
                converged = True
                break
        if config.fixed_passes is not None and stats:
            converged = _is_converged(stats[-1], config)
        x, f = sess.state()
        duals = DualStore(instance.n, config.workers)
        keys, vals, pd = sess.duals()
        _fill_duals(duals, keys, vals, pd, sess, None if plan.kind == "serial" else plan.b, plan.p)
    finally:
        sess.close()
    return Solution(state=PrimalState(instance.n, x, f), stats=stats, converged=converged,
                    passes_run=len(stats), total_steps=total, duals=duals)


def kkt_report(instance, state, duals):
    """Fixed-point audit (solver.py:256-281): state relation
    c + A'y = -eps W v, dual positivity, exact violation, complementarity."""
    g = core.accumulate_aty(instance, duals)
    target = -instance.epsilon * np.concatenate([instance.reg_x * state.xv,
                                                 instance.reg_f * state.fv])
    scale = max(1.0, float(np.max(np.abs(target))))
    residual = float(np.max(np.abs(g - target))) / scale
    n, m = instance.n, instance.npairs
    v = state.v()
    comp = 0.0
    min_y = np.inf
    keys, vals = duals.metric_arrays()
    if len(keys):
        i, j, k, kind = core.decode_keys(keys, n)
        pij = i * (n - 1) - i * (i - 1) // 2 + (j - i - 1)
        pik = i * (n - 1) - i * (i - 1) // 2 + (k - i - 1)
        pjk = j * (n - 1) - j * (j - 1) // 2 + (k - j - 1)
        plus = np.where(kind == 0, pij, np.where(kind == 1, pik, pjk))
        m1 = np.where(kind == 0, pik, pij)
        m2 = np.where(kind == 2, pik, pjk)
        av = v[plus] - v[m1] - v[m2]
        comp = max(comp, float(np.max(vals * np.maximum(-av, 0.0))))
        min_y = min(min_y, float(np.min(vals)))
    pu, pl = duals.pair_duals[:, 0], duals.pair_duals[:, 1]
    d = instance.d_flat
    au = state.xv - state.fv
    al = -state.xv - state.fv
    for y, a, rhs in ((pu, au, d), (pl, al, -d)):
        nz = y != 0.0
        if np.any(nz):
            comp = max(comp, float(np.max(y[nz] * np.maximum(rhs[nz] - a[nz], 0.0))))
            min_y = min(min_y, float(np.min(y[nz])))
    return {
        "state_relation_residual": residual,
        "min_stored_dual": float(min_y) if np.isfinite(min_y) else None,
        "max_violation": core.max_violation(instance, state),
        "complementary_slackness": comp,
    }
