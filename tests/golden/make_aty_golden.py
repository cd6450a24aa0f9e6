"""Golden vectors for c + A^T y (core.accumulate_aty, core.py:285-293) and the
dual objective (core.py:320-327), produced by the UNMODIFIED reference.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_aty_golden.py     # writes tests/golden/aty.npz

Cases: (1) a random store on n = 24 (two workers, random pair duals, zeros
included); (2) the reference's own duals after 6 tiled passes of config 1
(n = 100), so the fixture carries realistic key order and magnitudes.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as mg  # noqa: E402  (reference copy + import set-up)

from paper_1901_10084_b200 import instances  # noqa: E402

rcore, rsolver = mg.rcore, mg.rsolver


def store_arrays(duals):
    keys = np.concatenate(duals.keys) if duals.keys else np.empty(0, np.int64)
    vals = np.concatenate(duals.vals) if duals.vals else np.empty(0)
    return keys.astype(np.int64), vals.astype(np.float64), duals.pair_duals.copy()


def main():
    out = {}
    # case 1: random store
    n = 24
    inst = instances.random_instance(n, seed=7)
    rinst = mg.ref_instance(inst)
    rng = np.random.default_rng(11)
    trip = rng.choice(n, size=(400, 3))
    trip = np.sort(trip, axis=1)
    trip = trip[(trip[:, 0] < trip[:, 1]) & (trip[:, 1] < trip[:, 2])]
    codes = ((trip[:, 0] * n + trip[:, 1]) * n + trip[:, 2]) * 3 + rng.integers(0, 3, len(trip))
    codes = np.unique(codes)
    rng.shuffle(codes)
    vals = rng.uniform(1e-3, 2.0, len(codes))
    d = rcore.DualStore(n, 2)
    h = len(codes) // 2
    d.keys = [codes[:h].astype(np.int64), codes[h:].astype(np.int64)]
    d.vals = [vals[:h], vals[h:]]
    m = n * (n - 1) // 2
    d.pair_duals = rng.uniform(0, 1, (m, 2)) * (rng.uniform(size=(m, 2)) < 0.4)
    k, v, pd = store_arrays(d)
    out.update(r_n=n, r_keys=k, r_vals=v, r_pd=pd, r_c=rinst.c_vector(),
               r_g=rcore.accumulate_aty(rinst, d), r_dual=rcore.dual_objective(rinst, d))
    # case 2: the reference's duals after 6 passes of config 1
    inst = instances.config_instance(1)
    rinst = mg.ref_instance(inst)
    cfg = rsolver.SolverConfig(workers=1, tile_size=40, schedule_kind="tiled", fixed_passes=6)
    sol = rsolver.solve(rinst, cfg)
    k, v, pd = store_arrays(sol.duals)
    out.update(c_n=inst.n, c_keys=k, c_vals=v, c_pd=pd, c_c=rinst.c_vector(),
               c_g=rcore.accumulate_aty(rinst, sol.duals),
               c_dual=rcore.dual_objective(rinst, sol.duals))
    np.savez_compressed(os.path.join(HERE, "aty.npz"), **out)
    print("wrote aty.npz:", len(out["r_keys"]), "random keys,", len(out["c_keys"]), "config-1 keys")


if __name__ == "__main__":
    main()
