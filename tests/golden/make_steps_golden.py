"""Fixtures for projection.dykstra_step (reference projection.py:63-87),
written by running the UNMODIFIED reference on seeded random rows.

    python tests/golden/make_steps_golden.py     # writes tests/golden/steps.npz

Each case: a random state (x, f), random reg_x / reg_f, a random key (all five
kinds), a random old dual (0 in a third of the cases, so the projection-only
branch is covered) and epsilon; the reference's state after the step, its
theta_plus and changed flag are stored.  Rows are applied in sequence on one
state per instance (each step sees the previous steps' writes).
"""

import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF, COPY = "/root/reference/pkg", "/tmp/metricproj_ref_copy"
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
if not os.path.isdir(COPY):
    shutil.copytree(REF, COPY)
sys.path.insert(0, os.path.join(COPY, "src"))

from metricproj import core as rcore, projection as rproj  # noqa: E402


def main():
    out = {}
    rng = np.random.default_rng(20261020)
    for case in range(6):
        n = int(rng.integers(3, 12))
        m = n * (n - 1) // 2
        D = np.zeros((n, n))
        D[np.triu_indices(n, 1)] = rng.integers(0, 2, m)
        D = D + D.T
        W = np.ones((n, n)) - np.eye(n)
        eps = float(rng.choice([0.2, 0.1, 0.7, 1.0 / 3.0]))
        reg_x = rng.uniform(0.3, 3.0, m) if case % 2 else None
        reg_f = rng.uniform(0.3, 3.0, m) if case % 2 else None
        inst = rcore.ProblemInstance(n, D, W, epsilon=eps, reg_x=reg_x, reg_f=reg_f)
        st = rcore.PrimalState(n, rng.normal(scale=0.6, size=m), rng.normal(scale=0.6, size=m))
        out[f"c{case}_n"] = np.array(n)
        out[f"c{case}_eps"] = np.array(eps)
        out[f"c{case}_D"] = D
        out[f"c{case}_regx"] = inst.reg_x.copy()
        out[f"c{case}_regf"] = inst.reg_f.copy()
        out[f"c{case}_x0"] = st.xv.copy()
        out[f"c{case}_f0"] = st.fv.copy()
        keys, ys, thetas, changed = [], [], [], []
        for _ in range(60):
            kind = int(rng.integers(0, 5))
            if kind <= 2:
                i, j, k = sorted(rng.choice(n, 3, replace=False))
                key = rcore.ConstraintKey(rcore.Kind(kind), int(i), int(j), int(k))
            else:
                i, j = sorted(rng.choice(n, 2, replace=False))
                key = rcore.ConstraintKey(rcore.Kind(kind), int(i), int(j))
            y = 0.0 if rng.random() < 0.33 else float(rng.exponential(0.5))
            o = rproj.dykstra_step(st, key, y, inst)
            keys.append([int(key.kind), key.i, key.j, key.k])
            ys.append(y)
            thetas.append(o.theta_plus)
            changed.append(o.changed)
        out[f"c{case}_keys"] = np.array(keys, dtype=np.int64)
        out[f"c{case}_y"] = np.array(ys)
        out[f"c{case}_theta"] = np.array(thetas)
        out[f"c{case}_changed"] = np.array(changed)
        out[f"c{case}_x1"] = st.xv.copy()
        out[f"c{case}_f1"] = st.fv.copy()
    path = os.path.join(HERE, "steps.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}")


if __name__ == "__main__":
    main()
