/*
 * metricproj_b200 -- C ABI of the B200-native Dykstra triangle sweep.
 *
 * Drop-in boundary for the hot path of the reference package `metricproj`
 * (arXiv 1901.10084).  The reference crosses from Python into native code at
 * four numba kernels that mutate caller-owned numpy arrays in place:
 *
 *   _kernels.metric_units_pass  (reference pkg/src/metricproj/_kernels.py:60-132)
 *   _kernels.serial_metric_pass (_kernels.py:135-183)
 *   _kernels.pair_pass          (_kernels.py:186-220)
 *   _kernels.max_violation      (_kernels.py:28-57)
 *
 * called once per (round, worker) from solver._worker_pass (solver.py:129-154)
 * and from core.max_violation (core.py:342-345).  Per-round host calls would
 * dominate on a GPU (about 2n/b rounds per pass), so this ABI moves the
 * boundary up to whole passes with device-resident state: one handle owns x,
 * f, the pair duals and the sparse metric duals on the GPU for a whole solve,
 * and `mp_run_passes` replaces the body of run_pass (solver.py:166-210).  The
 * exact scan keeps a kernel-level entry (`mp_max_violation`) with the same
 * host-buffer contract as `_kernels.max_violation`.
 *
 * Conventions
 *   - All host buffers are caller-owned; device memory is the library's.
 *   - Pair-indexed arrays use the reference's packed order: pair (i,j), i<j,
 *     at i*(n-1) - i*(i-1)/2 + (j-i-1)  (core.py:40-44, _kernels.py:23-25).
 *   - Metric dual keys use ConstraintKey.encode: ((i*n+j)*n+k)*3 + kind
 *     (core.py:81-85), kinds 0/1/2 = IJ/IK/JK (core.py:25-28).
 *   - Every function returns MP_OK (0) or an MP_ERR_* code; mp_last_error()
 *     gives a thread-local message.  No C++ exception crosses the ABI.
 *   - One host thread per handle at a time.
 *   - There is no CPU fallback: without a usable sm_100 device every
 *     compute entry fails with MP_ERR_CUDA.
 */
#ifndef METRICPROJ_B200_H
#define METRICPROJ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MP_OK 0
#define MP_ERR_ARG 1       /* bad argument (ValueError in the Python mirror)      */
#define MP_ERR_CUDA 2      /* CUDA runtime / device error                          */
#define MP_ERR_OOM 3       /* device allocation failed                             */
#define MP_ERR_NONFINITE 4 /* non-finite x or f after a pass (SolverError,          *
                            * solver.py:200-201)                                   */
#define MP_ERR_UNSUPPORTED 5 /* configuration the device path does not implement   */

#define MP_SCHEDULE_SERIAL 0   /* SolverConfig.schedule_kind "serial"   (solver.py:21) */
#define MP_SCHEDULE_DIAGONAL 1 /* "diagonal": tiled with b = 1          (solver.py:77) */
#define MP_SCHEDULE_TILED 2    /* "tiled" (default), tile size b        (solver.py:31) */

#define MP_FLAG_TIME_ROUNDS 1u /* record per-kernel CUDA events (metric vs pair phase) */

/* ProblemInstance (core.py:97-159) in packed form.  reg_x / reg_f may be NULL
 * for the identity regularizer (core.py:131-134). */
typedef struct {
    int64_t n;
    const double *d_flat; /* C(n,2) dissimilarities d_ij */
    const double *w_flat; /* C(n,2) pair weights w_ij    */
    const double *reg_x;  /* C(n,2) or NULL              */
    const double *reg_f;  /* C(n,2) or NULL              */
    double epsilon;       /* > 0                          */
} mp_instance;

/* The part of SolverConfig (solver.py:28-51) that shapes the sweep. */
typedef struct {
    int32_t schedule_kind; /* MP_SCHEDULE_* */
    int32_t tile_b;        /* tile size b >= 1 (ignored for diagonal) */
    int32_t device;        /* CUDA device ordinal */
    uint32_t flags;        /* MP_FLAG_* */
} mp_config;

/* PassStats (core.py:259-267) plus device-side bookkeeping. */
typedef struct {
    int64_t pass_index;
    int64_t steps;         /* 3*C(n,3) + 2*C(n,2) per pass (_kernels.py:130,206,219) */
    int64_t nnz_metric;    /* metric duals stored after this pass (DualStore.nnz)   */
    double primal_objective;
    double dual_objective;
    double duality_gap;
    double max_violation;  /* running max of pre-step row values, metric and pair  */
    double wall_time;      /* seconds, CUDA events around the pass on the device   */
} mp_pass_stats;

typedef struct mp_handle mp_handle;

/* Create a solver session: validates and uploads the instance, builds the
 * schedule (schedule.tiled_rounds, schedule.py:117-153) and the device
 * tables, and sets the Dykstra start x = 0, f = -w/(eps*reg_f), y = 0
 * (solver.initialize, solver.py:108-113). */
int mp_create(const mp_instance *inst, const mp_config *cfg, mp_handle **out);

/* Run npasses full Dykstra passes (run_pass, solver.py:166-210): all metric
 * rounds in schedule order, then the pair phase, then the objectives.  Fills
 * out[0..npasses).  Stops early with MP_ERR_NONFINITE (after filling that
 * pass's stats) if x or f became non-finite. */
int mp_run_passes(mp_handle *h, int32_t npasses, mp_pass_stats *out);

/* Copy the primal state (PrimalState.xv / .fv, core.py:162-176) out / in. */
int mp_get_state(mp_handle *h, double *xv, double *fv);
int mp_set_state(mp_handle *h, const double *xv, const double *fv);

/* Number of stored metric duals (DualStore.nnz, core.py:240-241). */
int64_t mp_dual_count(mp_handle *h);

/* Export the duals: metric keys/values in the reference's single-worker visit
 * order (what DualStore.keys[0]/vals[0] hold for workers=1, core.py:218-236),
 * and the dense pair duals [C(n,2)][2] (core.py:235).  keys/vals need
 * mp_dual_count() entries; any pointer may be NULL to skip that part. */
int mp_get_duals(mp_handle *h, int64_t *keys, double *vals, double *pair_duals);

/* Import duals (any order of keys; each must be a metric key of this n with
 * a value > 0).  pair_duals may be NULL to keep the current ones. */
int mp_set_duals(mp_handle *h, int64_t nnz, const int64_t *keys, const double *vals,
                 const double *pair_duals);

/* Exact maximum violation of the session's current state (core.max_violation,
 * core.py:342-345), computed on the device. */
int mp_state_max_violation(mp_handle *h, double *out);

/* Device kernel time of the last mp_run_passes call, split by phase, when the
 * session was created with MP_FLAG_TIME_ROUNDS; launches = kernels launched. */
int mp_get_timing(mp_handle *h, double *metric_ms, double *pair_ms, int64_t *launches);

/* Optional in-kernel cycle counters of the tile kernel (diagnostics):
 * enable != 0 turns them on for later passes; out (if non-NULL) receives up
 * to nslots counters accumulated since the last read and resets them. */
int mp_trace(mp_handle *h, int32_t enable, uint64_t *out, int32_t nslots);

/* Write a buffer larger than L2 on the session's stream (benchmark hygiene). */
int mp_flush_l2(mp_handle *h);

void mp_destroy(mp_handle *h);

/* Like mp_get_duals (metric part only), plus order[e] = schedule index of the
 * tile entry e belongs to.  On a sharded session it returns that shard's
 * duals; concatenating every shard's output and stable-sorting it by order
 * gives the single-worker visit order. */
int mp_get_duals_ranked(mp_handle *h, int64_t *keys, double *vals, int64_t *order);

/* ---- One instance over several GPUs ------------------------
 * Replaces the reference's worker threads (solver._worker_pass,
 * solver.py:116-163; round ownership Round.worker_of, schedule.py:79-80) with
 * one process per GPU.  The tiles of each round are assigned to ranks by
 * longest-processing-time (mp_shard_plan); a rank keeps a whole x, runs its
 * tiles, keeps their duals, and after every round sends each b x b block its
 * tiles wrote to the rank whose tile touches that block next (grouped NCCL
 * send/recv on the session stream; a block's last toucher of the pass sends it
 * to every rank), so every tile reads what a single GPU would hold and every
 * rank follows the single-GPU trajectory bit for bit.  Counters (nnz, max
 * violation) are all-reduced, so every rank reports the global PassStats. */

/* Tile owners of the LPT plan, in schedule order (host only, no device).
 * owner may be NULL to query the tile count. */
int mp_shard_plan(int64_t n, int32_t b, int32_t world, int32_t *owner, int64_t *ntiles);

/* 128-byte NCCL unique id (rank 0 creates it, the caller broadcasts it). */
int mp_nccl_unique_id(void *id);

/* Make a fresh session (before its first pass) rank `rank` of `world`.  With
 * nccl_id != NULL the ranks are processes joined by an NCCL communicator
 * (blocks until all ranks call it) and mp_run_passes runs the sharded pass.
 * With nccl_id == NULL the session is a member of a local group: several
 * sessions of one process driven together by mp_group_run_passes (exchange by
 * device copies; a test transport that shares the exact per-round code). */
int mp_shard(mp_handle *h, int32_t world, int32_t rank, const void *nccl_id);

/* Values (8 bytes each, padding included) this rank sends and receives per
 * pass under the exchange plan of mp_shard (0 for an unsharded session). */
int mp_shard_volume(mp_handle *h, int64_t *sent, int64_t *received);

/* The exchange plan of a `world`-way sharded solve (host only, no device):
 * vol[(r * world + src) * world + dst] = pairs rank src sends to rank dst
 * after round r.  vol may be NULL to query the round count. */
int mp_shard_route(int64_t n, int32_t b, int32_t world, int64_t *vol, int64_t *nrounds);

/* Run npasses over a local group (hs[0..world) = the local shards, any order);
 * out[] receives the (global) stats, identical on every member. */
int mp_group_run_passes(mp_handle *const *hs, int32_t world, int32_t npasses, mp_pass_stats *out);

/* Kernel-level drop-in for _kernels.max_violation(xv, fv, dflat, n)
 * (_kernels.py:28-57): host buffers in, exact max violation out.  Runs on the
 * current CUDA device. */
int mp_max_violation(int64_t n, const double *xv, const double *fv, const double *d_flat,
                     double *out);

/* Kernel-level drop-in for core.accumulate_aty(instance, duals)
 * (core.py:285-293): g = c + A^T y over the stored duals, host buffers in and
 * out.  keys[nnz] = ConstraintKey.encode codes (core.py:81-85) with vals[nnz]
 * in DualStore.items() order; pair_duals = [C(n,2)][2] (upper, lower);
 * c = instance.c_vector() (length 2 C(n,2)); g receives 2 C(n,2) values, bit
 * for bit the reference's sequential accumulation (per target, contributions
 * in items() order).  Runs on the current CUDA device; invalid key ->
 * MP_ERR_ARG. */
int mp_accumulate_aty(int64_t n, int64_t nnz, const int64_t *keys, const double *vals,
                      const double *pair_duals, const double *c, double *g);

/* Kernel-level drop-in for projection.dykstra_step(state, key, y_old, instance)
 * (projection.py:63-87), batched: rows r = 0..nrows-1 are applied in order to
 * the value vector v[nv] (host buffer, updated in place).  Row r has nent[r]
 * entries (3 metric, 2 pair): positions pos[3r+e] into v, coefficients
 * coef[3r+e] (+-1, core._row_entries), weights reg[3r+e] (reg_x or reg_f of
 * the entry), right-hand side rhs[r] and old dual y_old[r] >= 0 (negative ->
 * MP_ERR_ARG, the reference's ValueError).  theta[r] receives theta_plus
 * (0 when <= THETA_FLOOR), changed[r] whether any entry moved.  Runs on the
 * current CUDA device, in dykstra_step's own association. */
int mp_dykstra_steps(int64_t nrows, const int32_t *nent, const int64_t *pos, const double *coef,
                     const double *reg, const double *rhs, const double *y_old, double eps,
                     int64_t nv, double *v, double *theta, int32_t *changed);

/* Correlation-clustering instance of a graph (instance.cc_instance,
 * instance.py:124-161): closed-neighbourhood Jaccard J of every pair (the
 * sparse product B*B^T on the device), s = log((1 + J - guard) / (1 - J +
 * guard)) clipped to [-cap, cap] and pushed off zero by `offset`; d = 1 where
 * s < 0 else 0, w = |s|, packed pair order.  The graph is CSR (rowptr[n+1],
 * cols[rowptr[n]]: sorted neighbour lists, no self-loops).  d is exact; w
 * matches numpy within the device log's accuracy (1 ulp). */
int mp_cc_instance(int64_t n, const int64_t *rowptr, const int32_t *cols, double guard, double cap,
                   double offset, double *d_flat, double *w_flat);

/* Self-test of the device's fast exact division (Markstein step with a
 * precomputed reciprocal, used for the divisions by eps and by 3 in the metric
 * step): compares it with IEEE division on `samples` random dividends and
 * reports the number of results that differ (must be 0). */
int mp_check_division(double divisor, int64_t samples, uint64_t seed, int64_t *mismatches);

/* Thread-local message for the last error on this thread ("" if none). */
const char *mp_last_error(void);

/* Library version string. */
const char *mp_version(void);

#ifdef __cplusplus
}
#endif

#endif /* METRICPROJ_B200_H */
