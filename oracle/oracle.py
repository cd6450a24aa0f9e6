"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the Dykstra triangle sweep.

Two restatements of the reference's hot path (arXiv 1901.10084 reference
package ``metricproj``), used only by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (``cpu_baseline`` and ``--impl reference``) as the checker /
CPU baseline.  The product (``paper_1901_10084_b200``) never imports this.

* :class:`OracleSolver` drives ``libmetricproj_oracle.so`` (``metricproj_oracle.c``,
  a C port of ``_kernels.py:28-220`` + ``solver.py:116-210``) and computes the
  per-pass objectives with numpy exactly as ``core.py:275-339`` does.
* :func:`py_pass` is a pure-Python loop restatement for tiny n, used to
  cross-check the C port inside the CPU test suite.

Parity is pinned: ``tests/golden/`` holds vectors produced by the unmodified
reference (``tests/golden/make_golden.py``); ``tests/test_oracle.py`` checks
both restatements against them bit for bit.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmetricproj_oracle.so")
THETA_FLOOR = 1e-15  # _kernels.py:20
KINDS = {"serial": 0, "diagonal": 1, "tiled": 2}

_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle in place (``make -C oracle``)."""
    src = os.path.join(HERE, "metricproj_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        D = ctypes.POINTER(ctypes.c_double)
        I = ctypes.POINTER(ctypes.c_int64)
        L.mpo_create.restype = P
        L.mpo_create.argtypes = [ctypes.c_int64, D, D, D, ctypes.c_double, ctypes.c_int,
                                 ctypes.c_int64, ctypes.c_int]
        L.mpo_destroy.argtypes = [P]
        L.mpo_set_state.argtypes = [P, D, D]
        L.mpo_get_state.argtypes = [P, D, D]
        L.mpo_get_pair_duals.argtypes = [P, D]
        L.mpo_dual_count.restype = ctypes.c_int64
        L.mpo_dual_count.argtypes = [P]
        L.mpo_get_duals.argtypes = [P, I, D]
        L.mpo_run_pass.restype = ctypes.c_double
        L.mpo_run_pass.argtypes = [P, I]
        L.mpo_max_violation.restype = ctypes.c_double
        L.mpo_max_violation.argtypes = [D, D, D, ctypes.c_int64]
        L.mpo_num_rounds.restype = ctypes.c_int64
        L.mpo_num_rounds.argtypes = [P]
        L.mpo_num_tiles.restype = ctypes.c_int64
        L.mpo_num_tiles.argtypes = [P]
        L.mpo_get_schedule.argtypes = [P, I, I]
        L.mpo_set_round_limit.argtypes = [P, ctypes.c_int64]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


@dataclass
class OracleStats:
    """Mirror of core.PassStats (core.py:259-267)."""
    pass_index: int
    primal_objective: float
    dual_objective: float
    duality_gap: float
    max_violation: float
    steps: int


def pair_count(n):
    return n * (n - 1) // 2


class OracleSolver:
    """Reference-order CPU solver over packed arrays (core.py layout)."""

    def __init__(self, n, d_flat, w_flat, eps, reg_x=None, reg_f=None,
                 kind="tiled", b=40, workers=1):
        m = pair_count(n)
        self.n, self.m, self.eps = n, m, float(eps)
        self.d_flat = np.ascontiguousarray(d_flat, dtype=np.float64)
        self.w_flat = np.ascontiguousarray(w_flat, dtype=np.float64)
        self.reg_x = np.ones(m) if reg_x is None else np.ascontiguousarray(reg_x, dtype=np.float64)
        self.reg_f = np.ones(m) if reg_f is None else np.ascontiguousarray(reg_f, dtype=np.float64)
        self.kind, self.b, self.workers = kind, b, workers
        L = lib()
        self._h = L.mpo_create(n, _dp(self.d_flat), _dp(self.reg_x), _dp(self.reg_f),
                               self.eps, KINDS[kind], b, workers)
        if not self._h:
            raise ValueError("oracle rejected the configuration")
        # Dykstra start (solver.py:108-113): x = 0, f = -w / (eps * reg_f)
        x0 = np.zeros(m)
        f0 = -self.w_flat / (self.eps * self.reg_f)
        L.mpo_set_state(self._h, _dp(x0), _dp(f0))
        self.passes = 0

    def close(self):
        if getattr(self, "_h", None):
            lib().mpo_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def state(self):
        x = np.empty(self.m)
        f = np.empty(self.m)
        lib().mpo_get_state(self._h, _dp(x), _dp(f))
        return x, f

    def set_state(self, x, f):
        x = np.ascontiguousarray(x, dtype=np.float64)
        f = np.ascontiguousarray(f, dtype=np.float64)
        lib().mpo_set_state(self._h, _dp(x), _dp(f))

    def pair_duals(self):
        pd = np.empty((self.m, 2))
        lib().mpo_get_pair_duals(self._h, _dp(pd))
        return pd

    def duals(self):
        c = lib().mpo_dual_count(self._h)
        keys = np.empty(c, dtype=np.int64)
        vals = np.empty(c)
        if c:
            lib().mpo_get_duals(self._h, _ip(keys), _dp(vals))
        return keys, vals

    def schedule(self):
        L = lib()
        nr = L.mpo_num_rounds(self._h)
        nt = L.mpo_num_tiles(self._h)
        rn = np.empty(nr, dtype=np.int64)
        xz = np.empty((nt, 2), dtype=np.int64)
        L.mpo_get_schedule(self._h, _ip(rn), _ip(xz))
        return rn, xz

    def timed_rounds(self, limit):
        """Timing sample only (bench.py's P = 1 row): run the first ``limit``
        rounds of one pass (no pair phase) and return (metric rows visited,
        seconds).  The solver is left mid-pass; close it afterwards."""
        import time
        L = lib()
        L.mpo_set_round_limit(self._h, int(limit))
        steps = ctypes.c_int64(0)
        t0 = time.perf_counter()
        L.mpo_run_pass(self._h, ctypes.byref(steps))
        dt = time.perf_counter() - t0
        L.mpo_set_round_limit(self._h, 0)
        return steps.value, dt

    def run_pass(self):
        steps = ctypes.c_int64(0)
        viol = lib().mpo_run_pass(self._h, ctypes.byref(steps))
        x, f = self.state()
        pd = self.pair_duals()
        primal, dual = objectives(self.eps, self.w_flat, self.d_flat, self.reg_x, self.reg_f, x, f, pd)
        st = OracleStats(self.passes, primal, dual, primal - dual, viol, steps.value)
        self.passes += 1
        return st


def objectives(eps, w_flat, d_flat, reg_x, reg_f, x, f, pd):
    """primal_objective (core.py:275-282) and dual_objective_from_state
    (core.py:330-339, with b_dot_y of core.py:314-317)."""
    lin = float(np.dot(w_flat, f))
    quad = float(np.dot(reg_x * x, x) + np.dot(reg_f * f, f))
    primal = lin + 0.5 * eps * quad
    bdy = float(np.dot(d_flat, pd[:, 0] - pd[:, 1]))
    dual = -bdy - 0.5 * eps * quad
    return primal, dual


def max_violation(x, f, d_flat, n):
    """Exact scan over all rows (_kernels.py:28-57)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    f = np.ascontiguousarray(f, dtype=np.float64)
    d = np.ascontiguousarray(d_flat, dtype=np.float64)
    return lib().mpo_max_violation(_dp(x), _dp(f), _dp(d), n)


# ---------------------------------------------------------------------------
# pure-Python restatement for tiny n (cross-check of the C port)
# ---------------------------------------------------------------------------

def _pos(n, i, j):
    return i * (n - 1) - i * (i - 1) // 2 + (j - i - 1)


def tiles_of(n, b):
    """tiled_rounds (schedule.py:117-153) as lists of (x, z)."""
    rounds = []

    def one(x, z):
        out, c = [], 0
        while max(x + c * b, 0) + 2 <= z - c * b:
            out.append((x + c * b, z - c * b))
            c += 1
        return out

    z = n - 1
    while z >= 2:
        rounds.append(one(1 - b, z))
        z -= b
    x = 1
    while x + 2 <= n - 1:
        rounds.append(one(x, n - 1))
        x += b
    return rounds


def tile_order(n, b, x, z):
    """Cube order of one tile (schedule.py:156-175)."""
    klo, ilo = max(z - b + 1, 0), max(x, 0)
    for jb in range(x + 1, z, b):
        je = min(jb + b - 1, z - 1)
        for k in range(klo, z + 1):
            for j in range(max(jb, 1), min(je, k - 1) + 1):
                for i in range(ilo, min(x + b - 1, j - 1) + 1):
                    yield (i, j, k)


def cube_order(n, c):
    """Serial order re-blocked into cubes of edge c: cube
    levels in increasing block sum I+J+K (I <= J <= K), the cubes of a level
    in any order (here: reversed, to show the order does not matter), and
    inside a cube the triplets level by level in L = i+j+k."""
    nb = (n + c - 1) // c
    for s in range(3 * nb):
        cubes = [(I, J, s - I - J) for I in range(nb) for J in range(I, nb)
                 if J <= s - I - J < nb]
        for (I, J, K) in reversed(cubes):
            trip = [(i, j, k) for i in range(I * c, min(n, I * c + c))
                    for j in range(max(J * c, i + 1), min(n, J * c + c))
                    for k in range(max(K * c, j + 1), min(n, K * c + c))]
            trip.sort(key=lambda t: (t[0] + t[1] + t[2], -t[0]))  # any order inside a level
            yield from trip


def visit_order(n, kind, b):
    if kind == "cube":
        yield from cube_order(n, b)
        return
    if kind == "serial":
        for i in range(n - 2):
            for j in range(i + 1, n - 1):
                for k in range(j + 1, n):
                    yield (i, j, k)
        return
    bb = 1 if kind == "diagonal" else b
    for rnd in tiles_of(n, bb):
        for (x, z) in rnd:
            yield from tile_order(n, bb, x, z)


def py_pass(n, eps, x, f, d_flat, winvx, winvf, duals, pair_duals, kind="tiled", b=40):
    """One pass in reference order; ``duals`` is a dict key->theta (the
    semantics of the cursor arrays), replaced by this pass's nonzero duals.
    Returns (viol, new_duals)."""
    viol = 0.0
    new = {}
    for (i, j, k) in visit_order(n, kind, b):
        pij, pik, pjk = _pos(n, i, j), _pos(n, i, k), _pos(n, j, k)
        code = ((i * n + j) * n + k) * 3
        for kd, (pl, m1, m2) in enumerate(((pij, pik, pjk), (pik, pij, pjk), (pjk, pij, pik))):
            y = duals.get(code + kd, 0.0)
            d0 = x[pl] - x[m1] - x[m2]
            if d0 > viol:
                viol = d0
            s = winvx[pl] + winvx[m1] + winvx[m2]
            delta = d0 + y * s / eps
            theta = eps * delta / s if delta > 0.0 else 0.0
            coef = (y - theta) / eps
            if coef != 0.0:
                x[pl] += coef * winvx[pl]
                x[m1] -= coef * winvx[m1]
                x[m2] -= coef * winvx[m2]
            if theta > THETA_FLOOR:
                new[code + kd] = theta
    for p in range(len(x)):
        d = d_flat[p]
        s = winvx[p] + winvf[p]
        for row in (0, 1):
            y = pair_duals[p, row]
            d0 = (x[p] - f[p] - d) if row == 0 else (d - x[p] - f[p])
            if d0 > viol:
                viol = d0
            delta = d0 + y * s / eps
            theta = eps * delta / s if delta > 0.0 else 0.0
            coef = (y - theta) / eps
            if coef != 0.0:
                if row == 0:
                    x[p] += coef * winvx[p]
                else:
                    x[p] -= coef * winvx[p]
                f[p] -= coef * winvf[p]
            pair_duals[p, row] = theta if theta > THETA_FLOOR else 0.0
    return viol, new


def dykstra_step_py(xv, fv, reg_x, reg_f, eps, n, kind, i, j, k, y_old, d_flat):
    """One row step in projection.dykstra_step's own association
    (projection.py:63-87): sums over the row's entries from 0, b last,
    W^-1 = 1/reg per entry.  Updates xv/fv in place; returns (theta, changed)."""
    m = pair_count(n)
    if kind <= 2:
        pij, pik, pjk = _pos(n, i, j), _pos(n, i, k), _pos(n, j, k)
        plus, m1, m2 = ((pij, pik, pjk), (pik, pij, pjk), (pjk, pij, pik))[kind]
        ent = ((plus, 1.0), (m1, -1.0), (m2, -1.0))
        b = 0.0
    else:
        p = _pos(n, i, j)
        ent = ((p, 1.0 if kind == 3 else -1.0), (m + p, -1.0))
        b = float(d_flat[p]) if kind == 3 else -float(d_flat[p])
    vals = [xv[q] if q < m else fv[q - m] for q, _ in ent]
    winv = [1.0 / (reg_x[q] if q < m else reg_f[q - m]) for q, _ in ent]
    d0 = sum(c * v for (_, c), v in zip(ent, vals)) - b
    s = sum(c * c * w for (_, c), w in zip(ent, winv))
    delta = d0 + y_old * s / eps
    theta = eps * delta / s if delta > 0.0 else 0.0
    coef = (y_old - theta) / eps
    if coef != 0.0:
        for (q, c), w in zip(ent, winv):
            if q < m:
                xv[q] += coef * c * w
            else:
                fv[q - m] += coef * c * w
    return (0.0 if theta <= THETA_FLOOR else theta), coef != 0.0


# ---------------------------------------------------------------------------
# instance construction (reference instance.py:124-161), numpy restatement
# ---------------------------------------------------------------------------

def cc_instance_np(rowptr, cols, n, offset=0.01, guard=0.05, cap=10.0):
    """Packed (d, w) of the signed Jaccard instance: closed neighbourhoods
    B (n x n, 0/1 with unit diagonal), inter = B B^T, union = |N[i]| + |N[j]|
    - inter, J = inter/union, s = log((1 + J - guard)/(1 - J + guard)),
    clip, offset away from 0; d = s < 0, w = |s| (instance.py:124-161)."""
    B = np.zeros((n, n))
    for u in range(n):
        B[u, cols[rowptr[u]:rowptr[u + 1]]] = 1.0
        B[u, u] = 1.0
    inter = B @ B.T
    sizes = B.sum(axis=1)
    union = sizes[:, None] + sizes[None, :] - inter
    J = inter / union
    s = np.log((1.0 + J - guard) / (1.0 - J + guard))
    np.clip(s, -cap, cap, out=s)
    s = np.where(s >= 0, s + offset, s - offset)
    iu = np.triu_indices(n, 1)
    return np.where(s < 0, 1.0, 0.0)[iu], np.abs(s)[iu]


def accumulate_aty_loop(n, keys, vals, pair_duals, c):
    """c + A^T y exactly as core.accumulate_aty (core.py:285-293) does it:
    ``DualStore.items()`` order (metric keys in store order, then the pair
    duals upper/lower per pair, core.py:244-253), each row's entries in
    ``_row_entries`` order (core.py:296-311), ``g[pos] += coef * y``.  Pure
    Python: tiny n only."""
    g = np.array(c, dtype=np.float64, copy=True)
    m = pair_count(n)
    for code, y in zip(keys, vals):
        code = int(code)
        kind, t3 = code % 3, code // 3
        i, j, k = t3 // (n * n), (t3 // n) % n, t3 % n
        pij, pik, pjk = _pos(n, i, j), _pos(n, i, k), _pos(n, j, k)
        ent = {0: ((pij, 1.0), (pik, -1.0), (pjk, -1.0)),
               1: ((pik, 1.0), (pij, -1.0), (pjk, -1.0)),
               2: ((pjk, 1.0), (pij, -1.0), (pik, -1.0))}[kind]
        for pos, coef in ent:
            g[pos] += coef * float(y)
    for p in range(m):
        yu, yl = float(pair_duals[p, 0]), float(pair_duals[p, 1])
        if yu != 0.0:
            g[p] += 1.0 * yu
            g[m + p] += -1.0 * yu
        if yl != 0.0:
            g[p] += -1.0 * yl
            g[m + p] += -1.0 * yl
    return g


def accumulate_aty_np(n, keys, vals, pair_duals, c):
    """Vectorised restatement of :func:`accumulate_aty_loop` with the same
    per-position addition order: ``np.add.at`` is unbuffered and sequential,
    so feeding it the row entries interleaved key by key (3e, 3e+1, 3e+2)
    reproduces the reference's loop bit for bit."""
    g = np.array(c, dtype=np.float64, copy=True)
    m = pair_count(n)
    keys = np.asarray(keys, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    if len(keys):
        kind, t3 = keys % 3, keys // 3
        i, j, k = t3 // (n * n), (t3 // n) % n, t3 % n
        rs = lambda a: a * (n - 1) - a * (a - 1) // 2  # noqa: E731
        pij, pik, pjk = rs(i) + j - i - 1, rs(i) + k - i - 1, rs(j) + k - j - 1
        plus = np.where(kind == 0, pij, np.where(kind == 1, pik, pjk))
        m1 = np.where(kind == 0, pik, pij)
        m2 = np.where(kind == 2, pik, pjk)
        tgt = np.stack([plus, m1, m2], axis=1).ravel()
        sv = np.stack([vals, -vals, -vals], axis=1).ravel()
        np.add.at(g, tgt, sv)
    yu, yl = pair_duals[:, 0], pair_duals[:, 1]
    gx, gf = g[:m], g[m:]
    nu, nl = yu != 0.0, yl != 0.0
    gx[nu] += yu[nu]
    gf[nu] += -yu[nu]
    gx[nl] += -yl[nl]
    gf[nl] += -yl[nl]
    return g
