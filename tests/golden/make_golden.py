"""Generate parity fixtures by running the UNMODIFIED reference solver.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_golden.py            # writes tests/golden/*.npz

The reference package is copied to /tmp (numba's cache=True would otherwise
write into the read-only reference tree) and imported from there.  Instances
come from paper_1901_10084_b200.instances (numpy only), so the tests can
rebuild them without the reference; the fixtures store hashes of the
instance vectors to catch generator drift.
"""

import hashlib
import os
import shutil
import sys
import time

import numpy as np

REF = "/root/reference/pkg"
COPY = "/tmp/metricproj_ref_copy"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
if not os.path.isdir(COPY):
    shutil.copytree(REF, COPY)
sys.path.insert(0, os.path.join(COPY, "src"))
sys.path.insert(0, os.path.join(COPY, "tests"))
sys.path.insert(0, ROOT)

from metricproj import core as rcore, solver as rsolver, projection as rproj  # noqa: E402
import reference as rref  # noqa: E402  (reference tests/reference.py: dense oracles)

from paper_1901_10084_b200 import instances  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_instance(inst):
    """Reference ProblemInstance with the same data."""
    n = inst.n
    D = np.zeros((n, n))
    W = np.zeros((n, n))
    iu = np.triu_indices(n, 1)
    D[iu] = inst.d_flat
    W[iu] = inst.w_flat
    D = D + D.T
    W = W + W.T
    return rcore.ProblemInstance(n, D, W, epsilon=inst.epsilon, reg_x=inst.reg_x.copy(),
                                 reg_f=inst.reg_f.copy())


def run_ref(rinst, kind, b, passes, workers, snap_passes=(), keep_duals_at=()):
    cfg = rsolver.SolverConfig(workers=workers, tile_size=b, schedule_kind=kind,
                               fixed_passes=passes)
    plan = rsolver.Plan(rinst.n, cfg)
    state, duals = rsolver.initialize(rinst, workers)
    pool = None
    if workers > 1:
        from concurrent.futures import ThreadPoolExecutor
        pool = ThreadPoolExecutor(max_workers=workers)
    rec = {k: [] for k in ("primal", "dual", "gap", "viol", "nnz", "xsha", "fsha", "steps")}
    snaps = {}
    t0 = time.time()
    for k in range(passes):
        st = rsolver.run_pass(state, duals, rinst, plan, pool=pool, pass_index=k)
        rec["primal"].append(st.primal_objective)
        rec["dual"].append(st.dual_objective)
        rec["gap"].append(st.duality_gap)
        rec["viol"].append(st.max_violation)
        rec["nnz"].append(duals.nnz())
        rec["steps"].append(st.steps)
        rec["xsha"].append(sha(state.xv))
        rec["fsha"].append(sha(state.fv))
        keys = np.concatenate(duals.keys) if duals.nnz() else np.empty(0, np.int64)
        vals = np.concatenate(duals.vals) if duals.nnz() else np.empty(0)
        rec.setdefault("dkeys_sha", []).append(sha(keys))
        rec.setdefault("dvals_sha", []).append(sha(vals))
        rec.setdefault("pd_sha", []).append(sha(duals.pair_duals))
        if (k + 1) in snap_passes:
            snaps[f"x_{k + 1}"] = state.xv.copy()
            snaps[f"f_{k + 1}"] = state.fv.copy()
        if (k + 1) in keep_duals_at:
            snaps[f"dkeys_{k + 1}"] = keys
            snaps[f"dvals_{k + 1}"] = vals
            snaps[f"pd_{k + 1}"] = duals.pair_duals.copy()
    if pool is not None:
        pool.shutdown()
    out = {k: np.array(v) for k, v in rec.items()}
    out.update(snaps)
    out["seconds"] = np.array(time.time() - t0)
    return out, state, duals


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")


def config_fixture(config, passes, workers, snap_passes, keep_duals_at, sample=None, n=None):
    inst = instances.config_instance(config, n=n)
    rinst = ref_instance(inst)
    out, state, duals = run_ref(rinst, "tiled", 40, passes, workers, snap_passes, keep_duals_at)
    meta = dict(config=np.array(config), n=np.array(inst.n), b=np.array(40),
                passes=np.array(passes), eps=np.array(inst.epsilon),
                dsha=np.array(sha(inst.d_flat)), wsha=np.array(sha(inst.w_flat)))
    if sample is not None:
        rng = np.random.default_rng(1234)
        idx = np.sort(rng.choice(inst.npairs, size=sample, replace=False))
        meta["sample_idx"] = idx
        meta["sample_x_final"] = state.xv[idx]
        meta["sample_f_final"] = state.fv[idx]
    meta["exact_viol_final"] = np.array(rcore.max_violation(rinst, state))
    return {**meta, **out}


def main(which):
    if "c1" in which:
        save("config1_n100_b40", **config_fixture(1, 50, 1, (2, 3, 50), ()))
    if "c2" in which:
        save("config2_n1000_b40_p4", **config_fixture(2, 4, 8, (), (), sample=4096))
    if "small" in which:
        small = {}
        rng = np.random.default_rng(7)
        cases = [(9, 2), (13, 3), (17, 5), (30, 8), (23, 4), (12, 1), (40, 40), (57, 16), (90, 40)]
        for n, b in cases:
            inst = instances.random_instance(n, seed=1000 + n)
            reg_x = rng.uniform(0.5, 2.0, inst.npairs)
            reg_f = rng.uniform(0.5, 2.0, inst.npairs)
            for wname, rx, rf in (("unit", None, None), ("reg", reg_x, reg_f)):
                rinst = ref_instance(inst)
                if rx is not None:
                    rinst.reg_x = rx.copy()
                    rinst.reg_f = rf.copy()
                out, state, duals = run_ref(rinst, "tiled", b, 6, 1, (6,), (6,))
                tag = f"n{n}_b{b}_{wname}"
                small[f"{tag}_x"] = state.xv
                small[f"{tag}_f"] = state.fv
                if n <= 30:
                    small[f"{tag}_pd"] = duals.pair_duals
                    small[f"{tag}_keys"] = out["dkeys_6"]
                    small[f"{tag}_vals"] = out["dvals_6"]
                small[f"{tag}_pdsha"] = np.array(sha(duals.pair_duals))
                small[f"{tag}_keysha"] = np.array(sha(out["dkeys_6"]))
                small[f"{tag}_valsha"] = np.array(sha(out["dvals_6"]))
                small[f"{tag}_nnz"] = out["nnz"]
                small[f"{tag}_viol"] = out["viol"]
                small[f"{tag}_primal"] = out["primal"]
                small[f"{tag}_dual"] = out["dual"]
                if rx is not None:
                    small[f"{tag}_regx"] = rx
                    small[f"{tag}_regf"] = rf
        # diagonal schedule
        inst = instances.random_instance(14, seed=77)
        rinst = ref_instance(inst)
        out, state, duals = run_ref(rinst, "diagonal", 1, 5, 1, (5,), (5,))
        small["diag_n14_x"] = state.xv
        small["diag_n14_f"] = state.fv
        small["diag_n14_keys"] = out["dkeys_5"]
        small["diag_n14_vals"] = out["dvals_5"]
        # serial schedule + the reference tests' dense Algorithm 1
        for n in (4, 5, 6, 9):
            inst = instances.random_instance(n, seed=100 * n)
            rinst = ref_instance(inst)
            out, state, duals = run_ref(rinst, "serial", 40, 3, 1, (3,), (3,))
            small[f"serial_n{n}_x"] = state.xv
            small[f"serial_n{n}_f"] = state.fv
            small[f"serial_n{n}_keys"] = out["dkeys_3"]
            small[f"serial_n{n}_vals"] = out["dvals_3"]
            if n <= 6:
                v, _ = rref.dense_dykstra(rinst, 3)
                small[f"dense_n{n}_v"] = v
        # exact violation scan on random states
        for n in (7, 31):
            inst = instances.random_instance(n, seed=n)
            rinst = ref_instance(inst)
            r = np.random.default_rng(n)
            st = rcore.PrimalState(n, r.normal(size=inst.npairs), r.normal(size=inst.npairs))
            small[f"scan_n{n}_x"] = st.xv
            small[f"scan_n{n}_f"] = st.fv
            small[f"scan_n{n}_viol"] = np.array(rcore.max_violation(rinst, st))
        # worked example (reference tests/test_acceptance.py:86-98)
        inst3 = rcore.ProblemInstance(3, np.zeros((3, 3)), np.ones((3, 3)) - np.eye(3), epsilon=0.7)
        st3 = rcore.PrimalState(3)
        st3.set_x(0, 1, 1.0)
        o = rproj.dykstra_step(st3, rcore.ConstraintKey(rcore.Kind.METRIC_IJ, 0, 1, 2), 0.0, inst3)
        small["worked_x"] = st3.xv
        small["worked_theta"] = np.array(o.theta_plus)
        save("small_cases", **small)


def graph_edges(seed):
    """Random edge lists with arbitrary node ids, a few duplicate and self-loop
    lines and a second, smaller component (seeded; written as text)."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(30, 160))
    p = float(rng.uniform(0.03, 0.15))
    ids = rng.permutation(10 * n)[:n] + 5
    e = [(ids[a], ids[b]) for a in range(n) for b in range(a + 1, n) if rng.random() < p]
    e += [e[t] for t in rng.integers(0, len(e), 3)]                # duplicates
    e += [(ids[t], ids[t]) for t in rng.integers(0, n, 2)]         # self loops
    base = 20 * n
    e += [(base + t, base + t + 1) for t in range(5)]              # small component
    rng.shuffle(e)
    return np.array(e, dtype=np.int64)


def graph_fixtures():
    """The reference's instance pipeline (instance.load_edge_list ->
    largest_component -> cc_instance) on seeded random edge lists."""
    from metricproj import instance as rinstance
    out = {}
    for seed in (3, 4, 5):
        edges = graph_edges(seed)
        path = f"/tmp/golden_graph_{seed}.txt"
        with open(path, "w") as fh:
            fh.write("# seeded random graph\n")
            for u, v in edges:
                fh.write(f"{u} {v}\n")
        g = rinstance.load_edge_list(path)
        comp = rinstance.largest_component(g)
        inst = rinstance.cc_instance(comp, epsilon=0.2)
        out[f"s{seed}_edges"] = edges
        out[f"s{seed}_n"] = np.array([g.n, comp.n, g.dropped_duplicates, g.dropped_self_loops])
        out[f"s{seed}_labels"] = np.array(comp.labels, dtype=np.int64)
        out[f"s{seed}_d"] = inst.d_flat
        out[f"s{seed}_w"] = inst.w_flat
    save("graphs", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "small", "c2", "graphs"]
    if "graphs" in which:
        graph_fixtures()
    main(which)
