"""Single-row Dykstra steps (reference ``projection.py``, same public names).

``dykstra_step`` is the reference's semantic definition of one step
(``projection.py:63-87``): correction with the old dual, projection, new
dual.  Here it runs on the GPU through ``mp_dykstra_steps`` (C ABI), in that
function's own association, so it returns the reference's values bit for
bit; the sweep kernels do the same step in bulk.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .core import _row_entries, pair_count


@dataclass(frozen=True)
class StepOutcome:
    """(projection.py:20-23)"""
    theta_plus: float
    changed: bool


def metric_row(key, n):
    """Positions, coefficients (+1, -1, -1) and b = 0 of a metric row
    (projection.py:26-35)."""
    if not key.is_metric:
        raise ValueError(f"not a metric key: {key}")
    entries = _row_entries(key, n)
    return tuple(p for p, _ in entries), tuple(c for _, c in entries), 0.0


def pair_row(key, instance):
    """Positions (one x, one f), coefficients and b = +d (upper) / -d (lower)
    of a pair row (projection.py:38-47)."""
    if key.is_metric:
        raise ValueError(f"not a pair key: {key}")
    entries = _row_entries(key, instance.n)
    return (tuple(p for p, _ in entries), tuple(c for _, c in entries), instance.rhs(key))


def constraint_row(key, instance):
    """(projection.py:50-53)"""
    if key.is_metric:
        return metric_row(key, instance.n)
    return pair_row(key, instance)


def dykstra_step(state, key, y_old, instance):
    """Correction with ``y_old``, projection and dual update for one
    constraint (projection.py:56-87).  Updates the 2 or 3 entries of
    ``state`` the row touches and returns the new dual and whether any
    variable moved."""
    from . import _native
    if y_old < 0:
        raise ValueError(f"dual values are nonnegative, got {y_old}")
    n = instance.n
    m = pair_count(n)
    positions, coeffs, b = constraint_row(key, instance)
    ne = len(positions)
    v = np.empty(ne)
    reg = np.ones(3)
    pos = np.zeros(3, dtype=np.int64)
    cf = np.zeros(3)
    for e, p in enumerate(positions):
        if p < m:
            v[e] = state.xv[p]
            reg[e] = instance.reg_x[p]
        else:
            v[e] = state.fv[p - m]
            reg[e] = instance.reg_f[p - m]
        pos[e] = e
        cf[e] = coeffs[e]
    nent = np.array([ne], dtype=np.int32)
    theta = np.zeros(1)
    changed = np.zeros(1, dtype=np.int32)
    L = _native.load()
    _native.check(L.mp_dykstra_steps(
        1, nent.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), _native.iptr(pos), _native.dptr(cf),
        _native.dptr(reg), _native.dptr(np.array([float(b)])), _native.dptr(np.array([float(y_old)])),
        float(instance.epsilon), ne, _native.dptr(v), _native.dptr(theta),
        changed.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))), "dykstra_step")
    if changed[0]:
        for e, p in enumerate(positions):
            if p < m:
                state.xv[p] = v[e]
            else:
                state.fv[p - m] = v[e]
    return StepOutcome(theta_plus=float(theta[0]), changed=bool(changed[0]))
