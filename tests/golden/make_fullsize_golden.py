"""Per-pass fixtures for BASELINE configs 2-5 at their full sizes.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_fullsize_golden.py c2 c3ref c3 c4 c5

* ``c2``    -- config 2 (n = 1000), all 100 passes, from the UNMODIFIED
  reference (imported from a /tmp copy, 8 workers; x is worker-independent
  because the tiles of a round are conflict-free, schedule.py:235-250).
* ``c3ref`` -- config 3 (n = 4000), passes 1-3 from the unmodified reference:
  pins the C oracle at this size (tests/test_oracle.py compares the two).
* ``c3``    -- config 3, all 200 passes, from the C oracle (all host threads;
  the reference would need ~2 h here).
* ``c4``    -- config 4 (n = 10000), passes 1-3, from the C oracle.
* ``c5``    -- config 5 (n = 18000), passes 1-3, from the C oracle.

Every pass records sha256 of x, f, the pair duals and the metric duals sorted
by reference key (``ConstraintKey.encode``, core.py:81-94) -- the sort makes
the hash independent of the worker count's store layout (core.py:218-236) --
plus max violation, nnz, steps and the objectives.  The GPU tests
(tests/test_gpu_golden_full.py) replay the same pass counts on the device and
compare every pass bit for bit.
"""

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_1901_10084_b200 import instances  # noqa: E402

B = 40


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def dual_sha(keys, vals):
    o = np.argsort(keys, kind="stable")
    return sha(np.asarray(keys, np.int64)[o]), sha(np.asarray(vals, np.float64)[o])


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)", flush=True)


def meta(config, inst, passes, source, workers):
    return dict(config=np.array(config), n=np.array(inst.n), b=np.array(B),
                passes=np.array(passes), eps=np.array(inst.epsilon),
                dsha=np.array(sha(inst.d_flat)), wsha=np.array(sha(inst.w_flat)),
                source=np.array(source), workers=np.array(workers))


def record(rec, x, f, pd, keys, vals, viol, nnz, steps, primal, dual):
    rec["xsha"].append(sha(x))
    rec["fsha"].append(sha(f))
    rec["pdsha"].append(sha(pd))
    ks, vs = dual_sha(keys, vals)
    rec["dkeys_sha"].append(ks)
    rec["dvals_sha"].append(vs)
    rec["viol"].append(viol)
    rec["nnz"].append(nnz)
    rec["steps"].append(steps)
    rec["primal"].append(primal)
    rec["dual"].append(dual)


def new_rec():
    return {k: [] for k in ("xsha", "fsha", "pdsha", "dkeys_sha", "dvals_sha", "viol", "nnz",
                            "steps", "primal", "dual")}


def finish(rec, state_x, state_f, extra):
    out = {k: np.array(v) for k, v in rec.items()}
    rng = np.random.default_rng(1234)
    idx = np.sort(rng.choice(len(state_x), size=min(4096, len(state_x)), replace=False))
    out["sample_idx"] = idx
    out["sample_x_final"] = state_x[idx]
    out["sample_f_final"] = state_f[idx]
    out.update(extra)
    return out


def run_reference(config, passes, workers=8):
    import shutil
    ref, copy = "/root/reference/pkg", "/tmp/metricproj_ref_copy"
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
    if not os.path.isdir(copy):
        shutil.copytree(ref, copy)
    sys.path.insert(0, os.path.join(copy, "src"))
    from concurrent.futures import ThreadPoolExecutor
    from metricproj import solver as rsolver
    sys.path.insert(0, HERE)
    from make_golden import ref_instance

    inst = instances.config_instance(config)
    rinst = ref_instance(inst)
    cfg = rsolver.SolverConfig(workers=workers, tile_size=B, schedule_kind="tiled",
                               fixed_passes=passes)
    plan = rsolver.Plan(rinst.n, cfg)
    state, duals = rsolver.initialize(rinst, workers)
    pool = ThreadPoolExecutor(max_workers=workers)
    rec = new_rec()
    t0 = time.time()
    for k in range(passes):
        st = rsolver.run_pass(state, duals, rinst, plan, pool=pool, pass_index=k)
        keys = np.concatenate(duals.keys) if duals.nnz() else np.empty(0, np.int64)
        vals = np.concatenate(duals.vals) if duals.nnz() else np.empty(0)
        record(rec, state.xv, state.fv, duals.pair_duals, keys, vals, st.max_violation,
               duals.nnz(), st.steps, st.primal_objective, st.dual_objective)
        print(f"ref config {config} pass {k + 1}/{passes} {time.time() - t0:.0f}s", flush=True)
    pool.shutdown()
    return inst, finish(rec, state.xv, state.fv,
                        {**meta(config, inst, passes, "reference", workers),
                         "seconds": np.array(time.time() - t0)})


def run_oracle(config, passes, workers=None):
    from oracle import oracle
    oracle.build()
    inst = instances.config_instance(config)
    workers = workers or int(os.environ.get("MP_GOLDEN_THREADS", 0)) or os.cpu_count() or 1
    ref = oracle.OracleSolver(inst.n, inst.d_flat, inst.w_flat, inst.epsilon, b=B,
                              workers=workers)
    rec = new_rec()
    t0 = time.time()
    for k in range(passes):
        st = ref.run_pass()
        x, f = ref.state()
        keys, vals = ref.duals()
        record(rec, x, f, ref.pair_duals(), keys, vals, st.max_violation, len(keys), st.steps,
               st.primal_objective, st.dual_objective)
        print(f"oracle config {config} pass {k + 1}/{passes} {time.time() - t0:.0f}s", flush=True)
    x, f = ref.state()
    ref.close()
    return inst, finish(rec, x, f, {**meta(config, inst, passes, "oracle", workers),
                                    "seconds": np.array(time.time() - t0)})


def main(which):
    if "c2" in which:
        _, out = run_reference(2, 100)
        save("full_config2_n1000_p100_ref", **out)
    if "c3ref" in which:
        _, out = run_reference(3, 3)
        save("full_config3_n4000_p3_ref", **out)
    if "c3" in which:
        _, out = run_oracle(3, 200)
        save("full_config3_n4000_p200_oracle", **out)
    if "c4" in which:
        _, out = run_oracle(4, 3)
        save("full_config4_n10000_p3_oracle", **out)
    if "c5" in which:
        _, out = run_oracle(5, 3)
        save("full_config5_n18000_p3_oracle", **out)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c3ref", "c3", "c4", "c5"])
