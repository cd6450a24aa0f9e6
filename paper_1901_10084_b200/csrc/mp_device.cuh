// Device side of the B200 Dykstra triangle sweep.
//
// Hot path: the reference's metric_units_pass (_kernels.py:60-132) executed
// for one round of conflict-free tiles (schedule.tiled_rounds,
// schedule.py:117-153) as ONE launch: one thread-block cluster of C CTAs per
// tile (CTA `band` owns tile rows [band*RB, band*RB + RB)), or one CTA per
// tile when a round has more tiles than clusters fit.
//
// Order exactness.  Two triplets conflict iff they share two indices; their
// index sums L = i+j+k then differ, and inside one round the reference's
// cube order (k, j, i ascending per j-chunk, _kernels.py:81-131) always
// visits the conflicting triplet with the smaller L first.
// Sweeping a tile level by level in L, any order inside a level, is
// therefore a linear extension of the reference order and reproduces its x
// bit for bit.  Thread slot (i,k) processes the triplet (i, L-i-k, k) at
// level L, all three rows in kind order IJ, IK, JK (_kernels.py:97-109).
// There are no per-level barriers: every conflict is ordered along the (i,k)
// lattice, so a warp only waits (per batch of MP_BATCH levels) for the warp
// holding its left columns and, in the previous band, the warp above it
// (see sweep()); warps of a band hold whole columns.
//
// Shared-memory layout of one tile (R = [ilo,ihi] rows i, K = [klo,z]
// columns k, J = [jlo,jhi] middle indices; SmemMap):
//   WR[rows][W]   x_ij, i in the band's rows, j in J, j < klo  -- ring over j
//   WK[W][b]      x_jk, j in J, j > ihi, k in K  -- ring over j, in x's row
//                 order (a 16-row block is one 2-D TMA box), replicated in
//                 every band, later bands receive exact-step writes by DSMEM
//   RK[b][b]      every pair (a,c) with a in R and c in K  (canonical home,
//                 so x_ij with j in K and x_jk with j in R alias into it)
// Row pitches of WR and WK are padded against bank conflicts (host-chosen).
// The rings are streamed from the dense (n x ld) x matrix in blocks of BLK
// j-values ahead of the fastest warp (TMA box + bulk row copies, or
// cp.async) and written back behind the slowest.  Each pair touched by a
// tile is touched by no other tile of the round (schedule.py:235-250), so no
// two clusters of a launch ever write the same x.
//
// Hot / cold split.  In the common case a row is neither violated nor has a
// stored dual, and the reference step is then a no-op (delta = d0 <= 0 ->
// theta = coef = 0).  The hot loop therefore only loads x_ij and x_jk (x_ik
// is register-held in the alias-free middle of a tile) and tests the rows
// with two DADDs; a batch with a violated row or a stored dual runs the exact
// reference step for the levels that need it (cold_batch / cold_slot).
//
// Arithmetic mirrors the reference bit for bit: explicit __dadd_rn /
// __dsub_rn / __dmul_rn and IEEE-exact division (no FMA contraction) in the
// reference's association (_kernels.py:115-125).  When W = I (reg_x == 1)
// the weights are exactly 1.0 and s = (1+1)+1 = 3 exactly, so the UNIT
// specialisation is bitwise identical to the general path.
//
// Sparse duals: each warp of each tile owns one "stream" of its nonzero
// duals, a linked list of 32-entry chunk records in a global pool.  Entries
// are (uint32 key, fp64 theta), key = ((L-Lbeg)*S + slot)*96 + lane*3 +
// kind, strictly increasing in the warp's own processing order, so the next
// pass replays them with a single warp cursor (the GPU analogue of the
// reference's per-worker cursor, _kernels.py:111-114).  The reader keeps
// the current and the next chunk in shared memory, the next one in flight
// as a bulk async copy (cp.async.bulk + mbarrier).  Values <= THETA_FLOOR
// are never stored (_kernels.py:126-129).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace mp {

// Checked builds (-DMP_CHECKED, tools/checked_tests.sh): device-side bounds
// and protocol assertions -- every shared-memory access inside the dynamic
// window, forwarded stores inside the replicated regions, dual-pool chunk
// indices below the pool capacity, dual keys strictly increasing per stream
// and never behind the read cursor, global ring addresses inside x, and
// dataflow predecessors claimed before their successors.  (compute-sanitizer
// is not available on this GPU pool; these checks stand in for it.)
#ifdef MP_CHECKED
#define MP_ASSERT(c)                                                                        \
    do {                                                                                    \
        if (!(c)) {                                                                         \
            printf("MP_ASSERT failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
                   (int)blockIdx.x, (int)threadIdx.x);                                      \
            __trap();                                                                       \
        }                                                                                   \
    } while (0)
#else
#define MP_ASSERT(c) \
    do {             \
    } while (0)
#endif

constexpr double THETA_FLOOR = 1e-15;  // _kernels.py:20
constexpr int BLK = 16;                // j-block width of the streamed rings
// levels per progress publish (batch) of a compute warp
#ifndef MP_BATCH
#define MP_BATCH 8
#endif
#ifndef MP_LOOKAHEAD  // ring blocks loaded ahead of the fastest compute warp
#define MP_LOOKAHEAD 4
#endif
#ifndef MP_OLD_PRODUCER  // 1: the cp.async producer also for TMA tiles (A/B only)
#define MP_OLD_PRODUCER 0
#endif
constexpr int CHUNK = 32;              // dual entries per pool chunk
constexpr uint32_t KEY_END = 0xFFFFFFFFu;
constexpr int MAX_CTA_THREADS = 512;   // >= 128 registers per thread
constexpr int MAX_SLOTS = 5;           // b <= 50 at 512 threads

struct TileDesc {
    int32_t ilo, ihi;    // rows i in [ilo, ihi]            (_kernels.py:76-77)
    int32_t klo, z;      // columns k in [klo, z]           (_kernels.py:78-80)
    int32_t jlo, jhi;    // middle j in [jlo, jhi]          (_kernels.py:81-86)
    int32_t Lbeg, Lend;  // level range of the tile, inclusive
    int64_t stream0;     // first warp-stream id of the tile
};

struct alignas(16) ChunkRec {
    uint32_t keys[CHUNK];  // KEY_END past the last entry
    double vals[CHUNK];
    int32_t next;          // next chunk of the stream, -1 at the end
    int32_t pad[3];
};
static_assert(sizeof(ChunkRec) == 400, "chunk record layout");

struct DualPool {
    ChunkRec *rec;  // [cap]
    int32_t *head;  // [nstreams] first chunk of each warp stream, -1 if empty
    int32_t cap;
};

struct PassCounters {
    unsigned long long viol_bits;  // atomicMax over non-negative doubles
    unsigned long long nnz;        // metric duals written this pass
    int32_t chunks_used;
    int32_t overflow;
    int32_t nonfinite;
    int32_t pad;
};

// Divisors of the metric step: eps (always) and s = 3 (W = I).
struct StepConsts {
    double eps, reps;  // eps and RN(1/eps); reps = 0 disables the fast path
    double r3;         // RN(1/3)
};

struct TileArgs {
    double *x;            // dense n x ld, upper triangle
    const double *winvx;  // dense n x ld, 1/reg_x (general W only)
    int64_t ld;
    const TileDesc *tiles;  // this round's tiles
    int32_t b;
    int32_t nt;  // threads per CTA
    double eps;
    DualPool rp, wp;
    PassCounters *ctr;
    int32_t nwc;  // compute warps per CTA (the rest are ring producers)
    StepConsts kc;
    unsigned long long *trace;  // optional cycle counters (mp_trace), null = off
    int32_t round_id;           // schedule round of this launch
    int32_t lw;                 // active lanes per warp slot row (<= 32)
    int32_t colm;               // column-major slot map in each band
    int32_t tl_round;           // MP_TIMELINE builds: round whose tile tl_tile is traced
    int32_t tl_tile;
    const void *tmap;           // 2-D TMA descriptor of x (box wkp x BLK), null: element copies
    int32_t wkp;                // WK row pitch in doubles (>= b; the TMA box width)
    int32_t wrp;                // WR row pitch in doubles (>= W)
    int32_t tma_store;          // interior WK blocks of the last band may be box-stored
    // Row bands of a cluster: band d owns tile rows [bst[d], bst[d+1]) (uniform
    // RB-row bands, or a split balancing the hub rows' exact steps), with
    // blw[d] active lanes per warp slot row; rbmax = the most rows of a band.
    uint8_t bst[17];
    uint8_t blw[16];
    int32_t rbmax;
    // Dataflow launch (df = 1): all tiles of the schedule's second family in
    // one launch; each cluster claims the next tile (qctr) and waits, ring
    // block by ring block, for the write-backs of the two tiles whose pairs it
    // reads next (dep: {row predecessor, column predecessor}, -1 = none in
    // this launch), published per (tile, band) in prog.  See DF_* below.
    int32_t df;
    const int4 *dep;  // {row, column, diagonal predecessor, 0}
    int32_t *prog;
    int32_t *qctr;
};

// Dataflow launch (second family of tiled_rounds, schedule.py:117-153):
// tiles (x + c*b, z - c*b) of round s with x >= 1.  Every pair a tile (x, z)
// touches was last touched (in the reference order) either by a first-family
// tile -- done before this launch starts -- or by one of two tiles of the
// previous round: its row predecessor (x, z - b), same rows, whose x_ij rows
// it reads as its own x_ij (WR ring) and, for j in [klo - b, klo), whose RK
// block it reads; and its column predecessor (x - b, z), same columns, whose
// x_jk rows (WK ring) hold this tile's x_jk rows and its RK rows.  (Checked
// exhaustively by tools/df_deps.py against the per-pair last-toucher of the
// whole schedule.)  Near the diagonal (z - x = b + 1, rows and columns
// overlapping) a tile may also read pairs its row predecessor never touched,
// last touched by the diagonal predecessor (x - b, z - b): such a tile waits
// for that one to finish before it starts (dep.z).
// prog[t * C + band] = ring blocks below it written back
// by band `band` of tile t (WR rows of the band; the last band also WK),
// DF_DONE once the tile finished (RK rows and the last blocks too).
constexpr int DF_DONE = 0x3fffffff;

#ifdef MP_TILETIME
// Diagnostic per-tile timing (tools/tile_times.py): per (round, tile, band)
// 16 u64 slots: globaltimer at kernel start / after the prologue / after the
// sweep / at the end, then the sweep's cycle counters summed over the
// compute warps (TR_PRED_WAIT .. TR_COLD_CALLS order, see TraceSlot).
constexpr int TT_ROUNDS = 256, TT_TILES = 128, TT_BANDS = 8, TT_REC = 16;
constexpr size_t TT_SLOTS = (size_t)TT_ROUNDS * TT_TILES * TT_BANDS * TT_REC;
#endif
#ifdef MP_TIMELINE
// Diagnostic timeline (tools/timeline.py): per (band, warp, batch) the clock64
// values [wait start, work start, work end, cold flag, levels replayed, lookup,
// math, append cycles]; warp slot 15 of each band holds [clock64,
// globaltimer] at the sweep start and end.
constexpr int TL_MAXB = 512;
constexpr int TL_REC = 8;  // u64 per batch record
constexpr int TL_SLOTS = 8 * 16 * TL_MAXB * TL_REC;
#endif
#if defined(MP_TIMELINE) || defined(MP_TILETIME)
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

// trace slots (cycles summed over warps / CTAs; see tools/trace_pass.py)
enum TraceSlot {
    TR_PRED_WAIT = 0, TR_RING_WAIT, TR_HOT, TR_COLD, TR_RELEASE, TR_LEVELS, TR_COLD_CALLS,
    TR_PROLOGUE = 8, TR_LOOP, TR_EPILOGUE, TR_EPI_BLOCKS, TR_CTAS, TR_C_LOOKUP, TR_C_MATH,
    TR_C_APPEND, TR_NSLOTS = 16
};

// Per-warp dual-stream state, in shared memory.
struct alignas(16) WarpDuals {
    ChunkRec buf[2];               // current / next chunk of the read stream
    unsigned long long mbar[2];    // completion of the bulk copy into buf[b]
    uint32_t phase[2];             // parity to wait for next, per buffer
    int32_t cur, pos;              // current buffer, first unconsumed entry
    int32_t has_next;              // buf[cur^1] holds (or receives) the next chunk
    uint32_t head;                 // key of the next unconsumed entry
    int32_t wchunk, wfill;         // writer: pool index of wbuf[wcur] (-1 none, -2 dead), fill
    uint32_t wcount;               // entries written by this warp
    int32_t pad;
    ChunkRec wbuf[2];              // writer staging: the chunk being filled, the one in flight
    int32_t wcur, wpad[3];
};

// Per-CTA constants, in shared memory (read by the out-of-line code).
struct CtaConst {
    TileDesc T;
    double *x;
    const double *winvx;
    int64_t ld;
    double eps;
    DualPool rp, wp;
    PassCounters *ctr;
    unsigned long long *trace;
    StepConsts kc;
    int32_t b, nt, xsize;
    int32_t C, band, RB;  // cluster size, this CTA's row band, most rows of a band (WR staging)
    int32_t nwc;          // compute warps per CTA
    int32_t tl;           // MP_TIMELINE: this CTA records its timeline
    int32_t B32;          // shared address of the aligned staging base
    int32_t lw;           // active lanes per warp slot row
    int32_t colm;         // column-major slot map (cluster bands)
    uint32_t rep_lo;      // shared address of WK (replicated in every band)
    uint32_t zero_lo;     // ... of the zero row (end of WK)
    uint32_t rk_lo;       // ... of RK
    uint32_t rk_row_mul;  // ceil(2^32 / (8b)): RK byte offset -> row (umulhi)
    uint8_t bst[17];      // band row starts (relative to ilo), bst[C] >= b
    uint8_t blw[16];      // lanes per warp slot row of each band (full rows)
    uint8_t rowband[64];  // tile row (relative) -> band
    const void *tmap;     // TMA descriptor of x (WK blocks), or null
    int32_t tma_st;       // the tile's K is b wide: interior WK blocks are stored by TMA
    int32_t wkp;          // WK row pitch (doubles)
    int32_t wrp;          // WR row pitch (doubles)
    unsigned long long *tt;  // MP_TILETIME builds: this CTA's record, else null
    // dataflow launch: the predecessors' progress words this CTA waits on
    // (null: none), the first ring block needing the row predecessor
    // finished, and this CTA's own progress word (null: not a dataflow launch)
    const int32_t *dep_r, *dep_c, *dep_d;  // dep_d: band 0 of the diagonal predecessor
    int32_t r_fin_blk;
    int32_t *my_prog;
};

#ifndef MP_CMAX  // largest cluster (CTAs per tile) the host plans; > 8 is non-portable
#define MP_CMAX 8
#endif
// Forwarding of an exact step's x_jk write to the later bands that read it
// (a cluster CTA's x_ij and x_ik lie in its own rows, which no later band
// reads): a WK value is read by every later band, an RK value (row j of the
// tile) by the later bands up to the owner of row j.  The remote stores are
// independent, so they are unrolled (issued back to back).  Returns whether
// anything was forwarded.
__device__ __forceinline__ uint32_t mapa(uint32_t a, unsigned rank);
__device__ __forceinline__ void st_cluster_f64(uint32_t a, double v);
__device__ __forceinline__ bool forward_jk(const CtaConst *cc, uint32_t ue, double e) {
#ifdef MP_EXP_NOFWD
    return false;  // timing experiment only: results are wrong
#endif
    const int C = cc->C, band = cc->band;
    MP_ASSERT((ue >= cc->rep_lo && ue < cc->zero_lo) || (ue >= cc->rk_lo && ue < cc->rk_lo + 8u * (uint32_t)(cc->b * cc->b)) ||
              (ue < cc->rep_lo));  // WK, RK, or a WR value (not forwarded: dlast = band)
    int dlast = band;
    if (ue >= cc->rep_lo && ue < cc->zero_lo) {
        dlast = C - 1;
    } else if (ue >= cc->rk_lo) {
        const uint32_t row = __umulhi(ue - cc->rk_lo, cc->rk_row_mul);
        dlast = min(C - 1, (int)cc->rowband[row]);
    }
#pragma unroll
    for (int d = 1; d < MP_CMAX; ++d)  // (unrolled to the largest cluster the host plans)
        if (band + d <= dlast) st_cluster_f64(mapa(ue, (unsigned)(band + d)), e);
    return dlast > band;
}

// ---------------------------------------------------------------------------
// one metric row, reference association (_kernels.py:115-125)
// ---------------------------------------------------------------------------
// Divisions whose value is known exactly are skipped: with y = 0,
// y*s/eps = +0 and delta = d0 (+0), so d0 <= 0 means theta = coef = 0 (no
// move, nothing stored) -- the same values the reference computes.
// Correctly rounded a/b from rb = RN(1/b) (Markstein): q0 = RN(a*rb) is
// within one ulp of a/b, the residual a - q0*b is exact with an FMA, and one
// correction RN(q0 + r*rb) rounds correctly.  The host enables it only for
// divisors with 2^-60 <= |b| <= 2^60 whose significand is not all ones; then
// a dividend with 2^-900 <= |a| <= 2^900 keeps every intermediate normal, and
// anything else (0, subnormal, huge, inf, nan) takes IEEE division.  The range
// test reads only a, so it runs beside the multiply chain.  Verified bit for
// bit against __ddiv_rn by mp_check_division (tests/test_gpu_parity.py).
// IEEE division, out of line: one copy for every rarely taken slow path
// (keeps the exact step's code small enough to stay in the instruction cache)
__device__ __noinline__ double ddiv_ieee(double a, double b) { return __ddiv_rn(a, b); }

__device__ __forceinline__ double div_rn(double a, double b, double rb) {
    const double aa = fabs(a);
    const double q0 = __dmul_rn(a, rb);
    const double r = __fma_rn(-q0, b, a);
    const double q1 = __fma_rn(r, rb, q0);
    if (!(aa >= 0x1p-900 && aa <= 0x1p+900)) return ddiv_ieee(a, b);
    return q1;
}

__device__ __forceinline__ double div_eps(double a, const StepConsts &k) {
    return k.reps != 0.0 ? div_rn(a, k.eps, k.reps) : ddiv_ieee(a, k.eps);
}

// s = (w_plus + w_m1) + w_m2 of a row (_kernels.py:118); 3 exactly for W = I
template <bool UNIT>
__device__ __forceinline__ double row_s(double wp, double wm1, double wm2) {
    return UNIT ? 3.0 : __dadd_rn(__dadd_rn(wp, wm1), wm2);
}

// One metric row given its value d0 = (plus - m1) - m2 and yq = (y*s)/eps
// (any value when y = 0): the reference step (_kernels.py:115-125).  Returns
// whether x moved (coef != 0); theta goes to th.
template <bool UNIT>
__device__ __forceinline__ bool row_step(double &p, double &m1, double &m2, double wp, double wm1,
                                         double wm2, double y, double yq, double d0,
                                         const StepConsts &k, double &viol, double &th) {
    viol = d0 > viol ? d0 : viol;
    th = 0.0;
    if (y == 0.0 && !(d0 > 0.0)) return false;
    const double delta = y == 0.0 ? d0 : __dadd_rn(d0, yq);
    double theta = 0.0;
    if (delta > 0.0)
        theta = UNIT ? div_rn(__dmul_rn(k.eps, delta), 3.0, k.r3)
                     : ddiv_ieee(__dmul_rn(k.eps, delta), row_s<UNIT>(wp, wm1, wm2));
    th = theta;
    const double coef = div_eps(__dsub_rn(y, theta), k);
    if (coef == 0.0) return false;
    if (UNIT) {
        p = __dadd_rn(p, coef);
        m1 = __dsub_rn(m1, coef);
        m2 = __dsub_rn(m2, coef);
    } else {
        p = __dadd_rn(p, __dmul_rn(coef, wp));
        m1 = __dsub_rn(m1, __dmul_rn(coef, wm1));
        m2 = __dsub_rn(m2, __dmul_rn(coef, wm2));
    }
    return true;
}

// One row, formed in place at its turn (_kernels.py:115-125).
template <bool UNIT>
__device__ __forceinline__ double dykstra_row(double &p, double &m1, double &m2, double wp,
                                              double wm1, double wm2, double y,
                                              const StepConsts &k, double &viol) {
    const double d0 = __dsub_rn(__dsub_rn(p, m1), m2);
    const double yq = y != 0.0 ? div_eps(__dmul_rn(y, row_s<UNIT>(wp, wm1, wm2)), k) : 0.0;
    double th;
    row_step<UNIT>(p, m1, m2, wp, wm1, wm2, y, yq, d0, k, viol, th);
    return th;
}

// The three rows of triplet (i,j,k) in kind order IJ, IK, JK (_kernels.py:97-
// 109), p = x_ij, c = x_ik, e = x_jk, each formed from the current values.
template <bool UNIT>
__device__ __forceinline__ void step3(double &p, double &c, double &e, double wa, double wc,
                                      double we, const double (&y)[3], const StepConsts &k,
                                      double &viol, double (&th)[3]) {
    th[0] = dykstra_row<UNIT>(p, c, e, wa, wc, we, y[0], k, viol);  // x_ij <= x_ik + x_jk
    th[1] = dykstra_row<UNIT>(c, p, e, wc, wa, we, y[1], k, viol);  // x_ik <= x_ij + x_jk
    th[2] = dykstra_row<UNIT>(e, p, c, we, wa, wc, y[2], k, viol);  // x_jk <= x_ij + x_ik
}

__device__ __forceinline__ void atomic_max_nonneg(unsigned long long *addr, double v) {
    // v >= 0: IEEE bit patterns of non-negative doubles order like the values
    if (v > 0.0) atomicMax(addr, (unsigned long long)__double_as_longlong(v));
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}

// ---------------------------------------------------------------------------
// async copy primitives
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
// ---- thread-block cluster primitives (one tile over C SMs) -------------------
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cluster_size() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
// shared::cta address -> the same offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t a, unsigned rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_f64(uint32_t a, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void st_release_cluster(uint32_t a, int v) {
    asm volatile("st.release.cluster.shared::cluster.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_cluster(uint32_t a, int v) {
    asm volatile("st.relaxed.cluster.shared::cluster.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_relaxed_cluster(uint32_t a) {
    int v;
    asm volatile("ld.relaxed.cluster.shared::cluster.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
// Acquire of a flag in the cluster window.  Everything this kernel shares
// across CTAs lives in shared memory, so the acquire is restricted to
// shared::cluster (a plain ld.acquire.cluster also invalidates L1: CCTL.IVALL).
__device__ __forceinline__ int ld_acquire_cluster(uint32_t a) {
    int v;
    asm volatile("ld.relaxed.cluster.shared::cluster.b32 %0, [%1];\n\t"
                 "fence.acquire.sync_restrict::shared::cluster.cluster;"
                 : "=r"(v) : "r"(a) : "memory");
    return v;
}
// Release of this thread's earlier remote (DSMEM) stores to the cluster.
__device__ __forceinline__ void fence_cluster() {
#ifndef MP_EXP_NOFENCE
    asm volatile("fence.release.cluster;" ::: "memory");
#endif
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

#ifdef MP_CHECKED
extern __shared__ __align__(1024) unsigned char mp_dyn_smem[];
__device__ __forceinline__ void chk_sh(uint32_t a) {
    uint32_t sz;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(sz));
    const uint32_t lo = (uint32_t)__cvta_generic_to_shared(mp_dyn_smem);
    MP_ASSERT(a >= lo && a + 8u <= lo + sz && (a & 7u) == 0u);
}
#else
__device__ __forceinline__ void chk_sh(uint32_t) {}
#endif
// 32-bit shared-window addresses: the per-slot constants already hold the
// absolute address, so the hot loop issues LDS [R] with no base add
__device__ __forceinline__ double ld_sh(uint32_t a) {
    chk_sh(a);
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void st_sh(uint32_t a, double v) {
    chk_sh(a);
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}
__device__ __forceinline__ void cp_async8s(uint32_t s, const void *gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(uint32_t s, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
// 16-byte shared -> global copy through registers
__device__ __forceinline__ void st_global_v2(double *gp, uint32_t s) {
    double a, c;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(c) : "r"(s) : "memory");
    asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(gp), "d"(a), "d"(c) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }
__device__ __forceinline__ void cp_async_wait_2() { asm volatile("cp.async.wait_group 2;\n" ::); }

__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
}
// one elected lane: arm the barrier for `bytes` and start the bulk copy
__device__ __forceinline__ void bulk_load(void *dst, const void *src, unsigned bytes,
                                          unsigned long long *bar) {
    asm volatile("fence.proxy.async.shared::cta;\n" ::);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 2-D TMA box load into this CTA's shared memory, completing on `bar`
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const void *tmap, int c0, int c1,
                                            unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
// 2-D TMA box store from this CTA's shared memory (bulk async-group)
__device__ __forceinline__ void tma_store_2d(const void *tmap, int c0, int c1, uint32_t src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];\n\t"
                 "cp.async.bulk.commit_group;" ::"l"(tmap),
                 "r"(c0), "r"(c1), "r"(src)
                 : "memory");
}
// non-blocking test of an mbarrier phase
__device__ __forceinline__ bool mbar_test(unsigned long long *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    return ok != 0;
}
// bulk copy global -> own shared memory completing on `bar` (no expect_tx)
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, unsigned bytes, unsigned long long *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

// ---------------------------------------------------------------------------
// warp-stream reader (shared-memory staged, bulk-copy prefetch)
// ---------------------------------------------------------------------------
// The cursor of a warp's read and write streams lives in registers (every
// lane holds the same values; `wcidx`/`wnext` only matter in lane 0), so an
// exact step's dual lookup and append cost no shared-memory round trips or
// warp barriers for bookkeeping; only the chunk data is in shared memory.
struct DualRegs {
    uint32_t head;     // key of the next unconsumed entry, KEY_END when none
    int32_t pos;       // its index in buf[cur]
    int32_t cur;       // read buffer holding the current chunk
    uint32_t ph;       // bit b: parity of buf[b]'s next bulk-copy completion
    int32_t has_next;  // buf[cur ^ 1] holds (or is receiving) the next chunk
    int32_t wstate;    // writer: -1 nothing written yet, -2 dead (pool overflow), 0 active
    int32_t wfill;     // entries staged in wbuf[wcur]
    int32_t wcur;      // staging buffer being filled
    uint32_t wcount;   // entries written by this warp
    int32_t wcidx;     // lane 0: pool index of the chunk staged in wbuf[wcur]
    int32_t wnext;     // lane 0: pool index allocated ahead for the next chunk (-3: none yet)
#ifdef MP_CHECKED
    uint32_t wlast;    // last key appended (keys must increase strictly)
    int32_t wany;
#endif
};

// Start of a tile: load the stream's first chunk, prefetch the second.
__device__ __forceinline__ void rd_init(DualRegs &r, WarpDuals *w, const DualPool &p, int64_t stream,
                                        int lane) {
    if (lane == 0) {
        mbar_init(&w->mbar[0], 1);
        mbar_init(&w->mbar[1], 1);
        mbar_fence_init();
    }
    __syncwarp();
    r.ph = 0u;
    r.cur = 0;
    r.pos = 0;
    r.wstate = -1;
    r.wfill = 0;
    r.wcur = 0;
    r.wcount = 0u;
    r.wcidx = -1;
    r.wnext = -3;
#ifdef MP_CHECKED
    r.wlast = 0u;
    r.wany = 0;
#endif
    const int32_t c = p.head[stream];
    if (c >= 0) {
        if (lane == 0) bulk_load(&w->buf[0], &p.rec[c], sizeof(ChunkRec), &w->mbar[0]);
        mbar_wait(&w->mbar[0], 0u);
        r.ph = 1u;
        const int32_t nx = w->buf[0].next;
        r.has_next = nx >= 0;
        if (lane == 0 && nx >= 0) bulk_load(&w->buf[1], &p.rec[nx], sizeof(ChunkRec), &w->mbar[1]);
        r.head = w->buf[0].keys[0];
    } else {
        r.has_next = 0;
        r.head = KEY_END;
        r.pos = CHUNK;
    }
}

// Consume every entry with key in [bs, bs + 96) (one slot of one level);
// lane l receives y[kind] of its triplet.  Warp-collective, no loop over
// entries: keys are sorted by (lane, kind), so an entry's chunk index is the
// number of in-range entries before it, read off per-kind lane masks
// (3 REDUX + POPC) -- each lane then loads its own values.
__device__ __forceinline__ void rd_lookup1(DualRegs &r, WarpDuals *w, const DualPool &p, uint32_t bs,
                                           int lane, double (&y)[3]) {
    const uint32_t lim = bs + 96u;
#ifdef MP_TIMELINE
    if (lane == 0) w->wpad[2] += 1;
#endif
    MP_ASSERT(r.head >= bs);  // every earlier level's entries were consumed
    while (r.head < lim) {
        const ChunkRec &c = w->buf[r.cur];
        const uint32_t key = c.keys[lane];
        const bool in = lane >= r.pos && key < lim;  // keys >= head >= bs
        const uint32_t off = key - bs;
        const uint32_t t = (off * 0xAAABu) >> 17;  // off / 3 (exact for off < 2^15)
        const uint32_t kd = off - 3u * t;
        const uint32_t bit = in ? (1u << (t & 31u)) : 0u;
        const uint32_t T0 = __reduce_or_sync(0xffffffffu, kd == 0u ? bit : 0u);
        const uint32_t T1 = __reduce_or_sync(0xffffffffu, kd == 1u ? bit : 0u);
        const uint32_t T2 = __reduce_or_sync(0xffffffffu, kd == 2u ? bit : 0u);
        const uint32_t below = (1u << lane) - 1u;
        const int q = r.pos + __popc(T0 & below) + __popc(T1 & below) + __popc(T2 & below);
        const int h0 = (int)((T0 >> lane) & 1u), h1 = (int)((T1 >> lane) & 1u), h2 = (int)((T2 >> lane) & 1u);
        MP_ASSERT(!(h0 | h1 | h2) || q + h0 + h1 + h2 <= CHUNK);
        if (h0) y[0] = c.vals[q];
        if (h1) y[1] = c.vals[q + h0];
        if (h2) y[2] = c.vals[q + h0 + h1];
        r.pos += __popc(T0) + __popc(T1) + __popc(T2);
#ifdef MP_TIMELINE
        if (lane == 0) w->wpad[0] += __popc(T0) + __popc(T1) + __popc(T2);
#endif
        if (r.pos >= CHUNK) {  // the level continues in (or the stream ends with) the next chunk
            if (!r.has_next) {
                r.head = KEY_END;
                break;
            }
            const int nb = r.cur ^ 1;
#ifdef MP_TIMELINE
            const long long tw0 = clock64();
#endif
            mbar_wait(&w->mbar[nb], (r.ph >> nb) & 1u);
#ifdef MP_TIMELINE
            if (lane == 0) { w->wpad[1] += (int)(clock64() - tw0); w->wpad[2] += 1 << 16; }
#endif
            r.ph ^= 1u << nb;
            __syncwarp();  // every lane is done with buf[cur] before it is refilled
            r.cur = nb;
            r.pos = 0;
            const int32_t nx = w->buf[nb].next;
            r.has_next = nx >= 0;
            MP_ASSERT(nx < p.cap);
            if (lane == 0 && nx >= 0) bulk_load(&w->buf[nb ^ 1], &p.rec[nx], sizeof(ChunkRec), &w->mbar[nb ^ 1]);
        }
        r.head = w->buf[r.cur].keys[r.pos];
    }
}

// ---------------------------------------------------------------------------
// warp-stream writer: appends this pass's nonzero duals
// ---------------------------------------------------------------------------
// Entries are staged in a shared-memory chunk and a full chunk goes to the
// pool with one bulk copy (cp.async.bulk, async proxy): no scattered global
// stores on the exact-step path, and a later release fence does not wait for
// them.  Two staging buffers: one filling, one possibly still being read by
// its bulk copy.  From a stream's second chunk on, the pool index of the next
// chunk is allocated one chunk ahead, so the allocation's atomic round trip
// is off the exact-step path.
// every lane that wrote the staged chunk: make its writes visible to the
// async proxy; then (after __syncwarp) one lane issues the copy
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_store(void *gdst, const void *ssrc, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\t"
                 "cp.async.bulk.commit_group;"
                 ::"l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_wait_read_le1() {
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// A pool index checked against the capacity (lane 0; -1 on pool overflow).
__device__ __forceinline__ int32_t wr_check(int32_t c, const DualPool &p, PassCounters *ctr) {
    if (c >= p.cap) {
        atomicExch(&ctr->overflow, 1);
        c = -1;
    }
    return c;
}

__device__ __forceinline__ void wr_append(DualRegs &r, WarpDuals *w, const DualPool &p, PassCounters *ctr,
                                          int64_t stream, uint32_t base, int lane, double t0,
                                          double t1, double t2) {
#ifdef MP_EXP_NOAPPEND
    return;  // timing experiment only: results are wrong
#endif
    const bool h0 = t0 > THETA_FLOOR, h1 = t1 > THETA_FLOOR, h2 = t2 > THETA_FLOOR;
    const unsigned m0 = __ballot_sync(0xffffffffu, h0);
    const unsigned m1 = __ballot_sync(0xffffffffu, h1);
    const unsigned m2 = __ballot_sync(0xffffffffu, h2);
    if ((m0 | m1 | m2) == 0u || r.wstate == -2) return;
    if (r.wstate == -1) {  // first entry of the stream: its first chunk
        int32_t c = 0;
        if (lane == 0) {
            c = wr_check(atomicAdd(&ctr->chunks_used, 1), p, ctr);
            p.head[stream] = c;
            r.wcidx = c;
        }
        c = __shfl_sync(0xffffffffu, c, 0);
        if (c < 0) {
            r.wstate = -2;
            return;
        }
        r.wstate = 0;
    }
    const unsigned lt = (1u << lane) - 1u;
    const int before = __popc(m0 & lt) + __popc(m1 & lt) + __popc(m2 & lt);
    const int total = __popc(m0) + __popc(m1) + __popc(m2);
#ifdef MP_CHECKED
    {  // the smallest key of this append is above the stream's last one
        const uint32_t kmin = base + 3u * (uint32_t)(__ffs(m0 | m1 | m2) - 1);
        MP_ASSERT(!r.wany || kmin > r.wlast);
        const int hl = 31 - __clz((int)(m0 | m1 | m2));
        r.wlast = base + 3u * (uint32_t)hl + 2u;
        r.wany = 1;
    }
    MP_ASSERT(lane != 0 || (r.wcidx >= 0 && r.wcidx < p.cap));
#endif
    // positions fill + before .. in key order (lane, kind); a position >= 32
    // belongs to a later chunk: write the window, flush, move on
    const double th[3] = {t0, t1, t2};
    const bool hk[3] = {h0, h1, h2};
    int start = 0;  // stream position of wbuf[wcur][0], relative to this append
    while (true) {
        int e = r.wfill + before;
#pragma unroll
        for (int kd = 0; kd < 3; ++kd) {
            if (hk[kd]) {
                const int pos = e - start;
                if (pos >= 0 && pos < CHUNK) {
                    w->wbuf[r.wcur].keys[pos] = base + 3u * (uint32_t)lane + (uint32_t)kd;
                    w->wbuf[r.wcur].vals[pos] = th[kd];
                }
                ++e;
            }
        }
        if (r.wfill + total - start < CHUNK) break;
        // wbuf[wcur] is full: link it to the next chunk and send it
        int32_t nxt = 0;
        if (lane == 0) {
            nxt = wr_check(r.wnext != -3 ? r.wnext : atomicAdd(&ctr->chunks_used, 1), p, ctr);
            w->wbuf[r.wcur].next = nxt;  // -1 on overflow: the pass is redone anyway
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
            bulk_store(&p.rec[r.wcidx], &w->wbuf[r.wcur], sizeof(ChunkRec));
            bulk_wait_read_le1();  // the other buffer's copy has read it
            r.wcidx = nxt;
            // allocate the chunk after `nxt` now; the value is first read at the next flush
            r.wnext = nxt >= 0 ? atomicAdd(&ctr->chunks_used, 1) : -1;
        }
        nxt = __shfl_sync(0xffffffffu, nxt, 0);
        if (nxt < 0) {
            r.wstate = -2;
            return;
        }
        r.wcur ^= 1;
        start += CHUNK;
    }
    r.wfill += total - start;
    r.wcount += (uint32_t)total;
}

__device__ __forceinline__ void wr_finish(DualRegs &r, WarpDuals *w, const DualPool &p, PassCounters *ctr,
                                          int64_t stream, int lane) {
    if (lane == 0 && r.wcount) atomicAdd(&ctr->nnz, (unsigned long long)r.wcount);
    if (r.wstate == 0) {
        if (lane >= r.wfill) w->wbuf[r.wcur].keys[lane] = KEY_END;
        if (lane == 0) w->wbuf[r.wcur].next = -1;
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) bulk_store(&p.rec[r.wcidx], &w->wbuf[r.wcur], sizeof(ChunkRec));
    } else if (r.wstate == -1) {
        if (lane == 0) p.head[stream] = -1;
    }
    if (lane == 0) bulk_wait_all();
    __syncwarp();
}

// ---------------------------------------------------------------------------
// ring staging of the j-window
// ---------------------------------------------------------------------------
// Load (LOAD=true, cp.async) or write back (LOAD=false) j-block `blk` of the
// WR / WK rings for array `g` (x or winvx) into ring arrays `wr`, `wk`.
// Predicates select exactly the pairs this tile touches that live in the
// rings (see the layout note above); nothing else is read or written.
// A cluster CTA stages only the WR rows of its band, [r0, r1) relative to
// ilo (stored from row 0 of its WR), and every CTA stages the whole WK; with
// with_wk = false the WK part is skipped (write-back by the last band only).
template <int W, bool LOAD>
__device__ __forceinline__ void ring_block(const TileDesc &T, int b, int p, int pr, int64_t ld, double *g,
                                           double *wr, double *wk, int blk, int tid, int nt,
                                           int r0, int r1, bool with_wk) {
#ifdef MP_EXP_NOWB
    if (!LOAD) return;  // timing experiment only: results are wrong
#endif
#ifdef MP_EXP_NOLOAD
    return;  // timing experiment only: results are wrong
#endif
    const int j0 = blk * BLK;
    // WR: rows i in the band x 8 column pairs (j, j+1), j even: row-contiguous
    // on both sides and 16-byte aligned (ld and W are multiples of 32), so an
    // in-range pair is one 16-byte copy.  x_ij lives in WR iff
    // jlo <= j <= min(jhi, klo - 1) and i < j.
    {
        const int wlo = T.jlo, whi = min(T.jhi, T.klo - 1);
        const int nwr = (r1 - r0) * (BLK / 2);
        for (int e = tid; e < nwr; e += nt) {
            const int ii = e >> 3, j = j0 + ((e & 7) << 1);
            const int i = T.ilo + r0 + ii;
            const bool v0 = i <= T.ihi && j >= wlo && j <= whi && i < j;
            const bool v1 = i <= T.ihi && j + 1 >= wlo && j + 1 <= whi && i < j + 1;
            if (!(v0 | v1)) continue;
            const uint32_t s = smem_u32(wr + ii * pr + (j & (W - 1)));
            double *gp = g + (int64_t)i * ld + j;
            MP_ASSERT(i >= 0 && j >= 0 && j + 1 < ld + 1 && i < j + 1);
            if (v0 & v1) {
                if (LOAD) cp_async16(s, gp);
                else st_global_v2(gp, s);
            } else {
                if (LOAD) {
                    if (v0) cp_async8s(s, gp);
                    if (v1) cp_async8s(s + 8, gp + 1);
                } else {
                    if (v0) gp[0] = ld_sh(s);
                    if (v1) gp[1] = ld_sh(s + 8);
                }
            }
        }
    }
    if (!with_wk) return;
    // WK: 16 rows j x columns k in K, shared layout WK[j % W][k - klo] (row
    // pitch b, the same order as x, so a whole block is one 2-D TMA box; this
    // element path serves the blocks TMA does not).  A warp takes one row j,
    // lanes over k: contiguous on both sides.
    // x_jk lives in WK iff jlo <= j <= jhi, j > ihi, j < k <= z.
    const int lane = tid & 31, nw = nt >> 5;
    const int jvlo = max(T.jlo, T.ihi + 1);
    for (int rr = tid >> 5; rr < BLK; rr += nw) {
        const int j = j0 + rr;
        if (j < jvlo || j > T.jhi) continue;
        const uint32_t srow = smem_u32(wk + (j & (W - 1)) * p);
        double *grow = g + (int64_t)j * ld + T.klo;
        if (!LOAD && !((T.klo | p) & 1)) {  // write-back in 16-byte pairs (both sides aligned)
            for (int kk = 2 * lane; kk < b; kk += 64) {
                const int k = T.klo + kk;
                const bool v0 = k <= T.z && j < k, v1 = kk + 1 < b && k + 1 <= T.z && j < k + 1;
                if (v0 & v1) {
                    st_global_v2(grow + kk, srow + 8 * kk);
                } else {
                    if (v0) grow[kk] = ld_sh(srow + 8 * kk);
                    if (v1) grow[kk + 1] = ld_sh(srow + 8 * kk + 8);
                }
            }
            continue;
        }
        for (int kk = lane; kk < b; kk += 32) {
            const int k = T.klo + kk;
            if (k <= T.z && j < k) {
                if (LOAD) cp_async8s(srow + 8 * kk, grow + kk);
                else grow[kk] = ld_sh(srow + 8 * kk);
            }
        }
    }
}

// RK block: rows i in R (relative rows [r0, r1)), columns k in K, i < k.  A
// warp takes a row, lanes over k; with klo and b even, 16-byte pairs (both
// sides aligned: RK rows are b doubles, x rows ld).
template <bool LOAD>
__device__ __forceinline__ void rk_block(const TileDesc &T, int b, int64_t ld, double *g,
                                         double *rk, int tid, int nt, int r0, int r1) {
    const int lane = tid & 31, nw = nt >> 5;
    const bool pairs = !((T.klo | b) & 1);
    for (int ii = r0 + (tid >> 5); ii < r1; ii += nw) {
        const int i = T.ilo + ii;
        if (i > T.ihi) continue;  // warp-uniform
        double *grow = g + (int64_t)i * ld + T.klo;
        const uint32_t srow = smem_u32(rk + ii * b);
        if (pairs) {
            for (int kk = 2 * lane; kk < b; kk += 64) {
                const int k = T.klo + kk;
                const bool v0 = k <= T.z && i < k, v1 = kk + 1 < b && k + 1 <= T.z && i < k + 1;
                if (v0 & v1) {
                    if (LOAD) cp_async16(srow + 8 * kk, grow + kk);
                    else st_global_v2(grow + kk, srow + 8 * kk);
                } else {
                    if (v0) {
                        if (LOAD) cp_async8s(srow + 8 * kk, grow + kk);
                        else grow[kk] = ld_sh(srow + 8 * kk);
                    }
                    if (v1) {
                        if (LOAD) cp_async8s(srow + 8 * kk + 8, grow + kk + 1);
                        else grow[kk + 1] = ld_sh(srow + 8 * kk + 8);
                    }
                }
            }
        } else {
            for (int kk = lane; kk < b; kk += 32) {
                const int k = T.klo + kk;
                if (k <= T.z && i < k) {
                    if (LOAD) cp_async8s(srow + 8 * kk, grow + kk);
                    else grow[kk] = ld_sh(srow + 8 * kk);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// the tile kernel: one CTA = one tile of the round
// ---------------------------------------------------------------------------
// Shared-memory map (byte offsets from a 1024-aligned base):
//   [0, b*W*8)            WR rows (1024 B each for W = 128)
//   [b*W*8, 2*b*W*8)      WK rows
//   [2*b*W*8, +W*8)       ZERO row (dummy target of inactive slots)
//   then RK[b*b], then (general W) the same layout for 1/reg_x, then the
//   per-warp dual state.
// A slot's ring address is ((L - i - k) * 8 & (W*8 - 8)) times the row
// pitch (WK) or plus the row base (WR); both pitches are padded so that the
// lanes of a warp spread over the banks (the host picks them per round).
template <int W>
struct SmemMap {
    int b;
    int rb;  // WR rows staged by this CTA (its band; b without a cluster)
    int p;   // WK row pitch in doubles (>= b, chosen against bank conflicts)
    int pr;  // WR row pitch in doubles (>= W, likewise)
    static __device__ __host__ int up(int x) { return (x + 127) & ~127; }
    __device__ __host__ int wr() const { return 0; }
    __device__ __host__ int wk() const { return up(rb * pr * 8); }
    __device__ __host__ int zero() const { return wk() + W * p * 8; }
    __device__ __host__ int rk() const { return zero() + W * 8; }
    __device__ __host__ int xbytes() const { return up(rk() + b * b * 8); }
};

// Lanes per warp slot row of a band with fewer real rows than the launch's
// bands (the single-row tiles): the band's slots spread evenly over all its
// compute warps (a hub row's exact steps then fall on many warps).  The host
// encodes / decodes dual keys with the same map (mp_solver.cu).
__host__ __device__ inline int band_lanes(int lw, int nwc, int S, int rows, int rb, int b, bool colm) {
    if (!colm || rows >= rb) return lw;
    const int per = nwc * S;
    return max(1, min(lw, (rows * b + per - 1) / per));
}

template <int S>
struct SlotGeom {
    int ik8[S];       // (i + k) * 8
    int off[S];       // active iff (unsigned)(L - off) <= span
    unsigned span[S];
    int pik[S];       // byte offset of x_ik (RK) or of the zero row
    int wr[S];        // byte offset of WR row ii (or zero row)
    int wk[S];        // byte offset of WK column kk (or zero row)
    int wkm[S];       // WK row pitch in doubles (M.p), 0 for an inactive slot
    int rkr[S];       // RK byte offset of x_ij when j in K:  rkr + 8j
    int rkc[S];       // RK byte offset of x_jk when j in R:  8*b*j + rkc
    int zero;         // shared address of the zero row
};

__device__ __forceinline__ double lds64(const unsigned char *base, int off) {
    return *reinterpret_cast<const double *>(base + off);
}

// Violation test of one triplet without forming the three row values.
// For finite or infinite x, y: fl(x - y) > 0  <=>  x > y (round-to-nearest
// keeps the sign and gradual underflow never rounds a nonzero difference to
// 0; NaN compares false both ways).  With t = fl(a - c), fl(c - a) = -t, so
//   d0 = fl(t - e) > 0   <=>  t > e
//   d1 = fl(-t - e) > 0  <=>  -t > e        i.e. (d0 > 0 || d1 > 0) <=> |t| > e
//   d2 = fl(fl(e - a) - c) > 0  <=>  fl(e - a) > c
// Two DADDs and two DSETPs instead of five and three; returns 1 if violated.
__device__ __forceinline__ unsigned triplet_violated(double a, double c, double e) {
    unsigned r;
    asm("{\n\t.reg .pred p;\n\t.reg .f64 t, u;\n\t"
        "sub.rn.f64 t, %1, %2;\n\t"
        "sub.rn.f64 u, %3, %1;\n\t"
        "abs.f64 t, t;\n\t"
        "setp.gt.f64 p, t, %3;\n\t"
        "setp.gt.or.f64 p, u, %2, p;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(r)
        : "d"(a), "d"(c), "d"(e));
    return r;
}

// Hot part of one level: true when some slot of this thread has a violated
// row; the slots' byte offsets are left in pa/pc/pe for the cold path.
// Branch-free: inactive slots read the zero row (all row values 0).  With
// t = fl(a - c), u = fl(e - a):  (d0 > 0 || d1 > 0) <=> |t| > e  and
// d2 > 0 <=> u > c, exactly (see triplet_violated).
// Shared addresses of x_ij, x_ik, x_jk of this thread's S slots at level L
// (the zero row for a slot with no triplet at L).
template <int S, int W, bool ALIAS>
__device__ __forceinline__ void slot_addrs(const SlotGeom<S> &G, int L, int b, int ihi, int klo,
                                           int (&pa)[S], int (&pc)[S], int (&pe)[S]) {
    const int L8 = L * 8;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int j8 = L8 - G.ik8[s];
        const int jm = j8 & (W * 8 - 8);
        if (ALIAS) {
            const bool act = (unsigned)(L - G.off[s]) <= G.span[s];
            const int j = j8 >> 3;
            int a0 = j >= klo ? G.rkr[s] + j8 : jm + G.wr[s];
            int e0 = j <= ihi ? j * (8 * b) + G.rkc[s] : jm * G.wkm[s] + G.wk[s];
            pa[s] = act ? a0 : G.zero;
            pe[s] = act ? e0 : G.zero;
            pc[s] = act ? G.pik[s] : G.zero;
        } else {
            pa[s] = jm + G.wr[s];
            pe[s] = jm * G.wkm[s] + G.wk[s];
            pc[s] = G.pik[s];
        }
    }
}

template <int S, int W, bool ALIAS>
__device__ __forceinline__ bool level_hot(const unsigned char *sm, const SlotGeom<S> &G, int L,
                                          int b, int ihi, int klo, int (&pa)[S], int (&pc)[S],
                                          int (&pe)[S], const double (&xcr)[S]) {
    slot_addrs<S, W, ALIAS>(G, L, b, ihi, klo, pa, pc, pe);
    double xa[S], xc[S], xe[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        xa[s] = ld_sh(pa[s]);
        // alias-free levels: x_ik belongs to this thread alone, kept in a register
        xc[s] = ALIAS ? ld_sh(pc[s]) : xcr[s];
        xe[s] = ld_sh(pe[s]);
    }
    bool bad = false;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const double t = __dsub_rn(xa[s], xc[s]);
        const double u = __dsub_rn(xe[s], xa[s]);
        bad = bad | (fabs(t) > xe[s]) | (u > xc[s]);
    }
    return bad;
}

// Slot geometry of this thread: slot q = (warp*S + s)*lw + lane within the
// band [r0, r1) of the tile; row-major (i, k) = (ilo + r0 + q/b, klo + q%b),
// or column-major in a cluster band (a warp then covers a few columns of all
// the band's rows, so the warps of consecutive bands form a 2-D grid rather
// than one long chain).  A warp may use only lw < 32 lanes per slot row.
template <int S, int W>
__device__ __forceinline__ void slot_geom(SlotGeom<S> &G, const TileDesc &T, const SmemMap<W> &M,
                                          int B32, int b, int r0, int r1, int warp, int lane, int lw,
                                          bool colm) {
    const int rbc = r1 - r0;  // rows of this band
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int q = (warp * S + s) * lw + lane;  // lanes >= lw idle (fewer slots per warp)
        // row-major: q = (i - ilo - r0)*b + (k - klo); column-major (cluster
        // bands): q = (k - klo)*rbc + (i - ilo - r0)
        const int ii = colm ? r0 + q % max(rbc, 1) : r0 + q / b;
        const int kk = colm ? q / max(rbc, 1) : q - (q / b) * b;
        const int i = T.ilo + ii, k = T.klo + kk;
        const int js = max(i + 1, T.jlo), je = min(k - 1, T.jhi);
        const bool ok = lane < lw && q < (r1 - r0) * b && i <= T.ihi && k <= T.z && js <= je;
        G.ik8[s] = ok ? 8 * (i + k) : 0;
        G.off[s] = ok ? i + k + js : 0x3fffffff;
        G.span[s] = ok ? (unsigned)(je - js) : 0u;
        G.pik[s] = B32 + (ok ? M.rk() + 8 * (ii * b + kk) : M.zero());
        G.wr[s] = B32 + (ok ? M.wr() + (ii - r0) * M.pr * 8 : M.zero());
        G.wk[s] = B32 + (ok ? M.wk() + kk * 8 : M.zero());
        G.wkm[s] = ok ? M.p : 0;
        G.rkr[s] = B32 + (ok ? M.rk() + 8 * (ii * b - T.klo) : M.zero());
        G.rkc[s] = B32 + (ok ? M.rk() + 8 * (kk - T.ilo * b) : M.zero());
    }
    G.zero = B32 + M.zero();
}

// ---------------------------------------------------------------------------
// cold path: the exact reference step for the levels of a batch that need it
// ---------------------------------------------------------------------------
// Levels [first, Le] of the batch starting at L0, in order.  A level is
// replayed if the hot check flagged it (bit Lc-L0 of `flagged`), if it holds
// one of this warp's stored duals, or if an earlier level of this batch moved
// x (the hot check read values this warp has since changed; other warps'
// values were final before the batch started).  Per level: the duals of all S
// slots in one pass over the warp stream, the three rows of every slot that
// needs them (reference association, _kernels.py:115-125), and the new duals
// appended in key order.  Out of line: the hot loop keeps its registers.
// Exact step of one slot of one level for the whole warp (used with S > 1,
// where cold_batch's live state would not fit the registers).  pa/pc/pe are
// the slot's shared addresses (the zero row for inactive lanes).  Returns the
// updated violation; `fwd` is set if a value was forwarded to a later band.
#ifndef MP_SLOT_INLINE
#define MP_SLOT_INLINE __noinline__
#endif
template <int W, bool UNIT>
__device__ MP_SLOT_INLINE double cold_slot(const CtaConst *cc, WarpDuals *wd, DualRegs &dr, int warp,
                                         uint32_t base, int pa, int pc, int pe, double viol, bool &fwd) {
    const int lane = threadIdx.x & 31;
    double p = ld_sh(pa), c = ld_sh(pc), e = ld_sh(pe);
    double y[3] = {0.0, 0.0, 0.0};
    if (dr.head < base + 96u) rd_lookup1(dr, wd, cc->rp, base, lane, y);
    double th[3] = {0.0, 0.0, 0.0};
    const bool need = (fabs(__dsub_rn(p, c)) > e) | (__dsub_rn(e, p) > c) | (y[0] != 0.0) |
                      (y[1] != 0.0) | (y[2] != 0.0);
    if (need) {
        double wa = 1.0, wc = 1.0, we = 1.0;
        if (!UNIT) {
            const int xb = cc->xsize * 8;
            wa = ld_sh(pa + xb);
            wc = ld_sh(pc + xb);
            we = ld_sh(pe + xb);
        }
        step3<UNIT>(p, c, e, wa, wc, we, y, cc->kc, viol, th);
        st_sh(pa, p);
        st_sh(pc, c);
        st_sh(pe, e);
        const int C = cc->C, band = cc->band;
        if (C > 1 && band + 1 < C) fwd |= forward_jk(cc, (uint32_t)pe, e);
    }
    const int64_t stream = cc->T.stream0 + (int64_t)cc->band * cc->nwc + warp;
    if (__any_sync(0xffffffffu, (th[0] > THETA_FLOOR) | (th[1] > THETA_FLOOR) | (th[2] > THETA_FLOOR)))
        wr_append(dr, wd, cc->wp, cc->ctr, stream, base, lane, th[0], th[1], th[2]);
    return viol;
}

// One level replayed exactly (S > 1): per slot, if some lane of the warp has
// a violated row or the slot holds a stored dual, the out-of-line cold_slot.
template <int S, int W, bool UNIT, bool ALIAS>
__device__ __forceinline__ bool level_full(int L, uint32_t base0, const unsigned char *sm,
                                           const SlotGeom<S> &G, const CtaConst *cc, WarpDuals *wd,
                                           DualRegs &dr, int warp, int b, int ihi, int klo,
                                           double (&xcr)[S], double &viol, bool &fwd) {
    int pa[S], pc[S], pe[S];
    level_hot<S, W, ALIAS>(sm, G, L, b, ihi, klo, pa, pc, pe, xcr);
    bool moved = false;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const uint32_t bs = base0 + (uint32_t)(s * 96);
        const double a = ld_sh(pa[s]), c = ld_sh(pc[s]), e = ld_sh(pe[s]);
        const bool bad = (fabs(__dsub_rn(a, c)) > e) | (__dsub_rn(e, a) > c);
        if (__any_sync(0xffffffffu, bad) || dr.head < bs + 96u) {
            viol = cold_slot<W, UNIT>(cc, wd, dr, warp, bs, pa[s], pc[s], pe[s], viol, fwd);
            if (!ALIAS) xcr[s] = ld_sh(pc[s]);  // the exact step may move x_ik
            moved = true;
        }
    }
    return moved;
}

#ifndef MP_COLD_INLINE
#define MP_COLD_INLINE __forceinline__  // inlined: no call, registers allocated with the sweep (-2.7% at config 2)
#endif
template <int S, int W, bool UNIT, bool ALIAS, int U>
__device__ MP_COLD_INLINE double cold_batch(int L0, int first, int Le, unsigned flagged,
                                          const CtaConst *cc, WarpDuals *wd, DualRegs &dr, int warp,
                                          double viol, const SlotGeom<S> G) {
    const int lane = threadIdx.x & 31;
    const TileDesc &T = cc->T;
    const int b = cc->b, C = cc->C, band = cc->band;
    constexpr uint32_t PER_LEVEL = (uint32_t)(S * 96);
    const int64_t stream = T.stream0 + (int64_t)band * cc->nwc + warp;
    const StepConsts k = cc->kc;
    const int xb = cc->xsize * 8;  // winv staging mirrors the x layout (general W)
    const bool fwd_band = C > 1 && band + 1 < C;
    bool fwd = false;
    // Levels left to replay: bit Lc - L0 set when some lane's row at Lc is
    // violated.  After a level that moved x the later levels are re-checked
    // with the new values (the hot test, all of them at once) instead of being
    // replayed one by one -- a replayed level with no violated row and no
    // stored dual is a no-op in the reference.  The loop jumps from level to
    // level: the next one is the next flagged level or the next holding a
    // stored dual (the cursor's head key names its level).
    unsigned todo = flagged;
#ifdef MP_TIMELINE
    long long tq0 = clock64(), c_lk = 0, c_mt = 0, c_ap = 0, c_ld = 0, nlev = 0;
    __syncwarp();
    if (lane == 0) wd->wpad[0] = wd->wpad[1] = wd->wpad[2] = 0;
    __syncwarp();
#endif
    for (int Lc = first; Lc <= Le;) {
        const uint32_t base = (uint32_t)(Lc - T.Lbeg) * PER_LEVEL;
#ifdef MP_TIMELINE
        ++nlev;
        long long tq = clock64();
#endif
        int pa[S], pc[S], pe[S];
        slot_addrs<S, W, ALIAS>(G, Lc, b, T.ihi, T.klo, pa, pc, pe);
        bool moved = false;
#pragma unroll
        for (int s = 0; s < S; ++s) {  // slot by slot: keys are ordered by slot
            const uint32_t bs = base + (uint32_t)(s * 96);
            // the level's x loads go out before the lookup (independent)
            double p = ld_sh(pa[s]), c = ld_sh(pc[s]), e = ld_sh(pe[s]);
            double y[3] = {0.0, 0.0, 0.0};
            if (dr.head < bs + 96u) rd_lookup1(dr, wd, cc->rp, bs, lane, y);
#ifdef MP_TIMELINE
            { const long long t = clock64(); c_lk += t - tq; tq = t; }
#endif
            double th[3] = {0.0, 0.0, 0.0};
            double wa = 1.0, wc = 1.0, we = 1.0;
            if (!UNIT) {
                wa = ld_sh(pa[s] + xb);
                wc = ld_sh(pc[s] + xb);
                we = ld_sh(pe[s] + xb);
            }
            const bool need = (fabs(__dsub_rn(p, c)) > e) | (__dsub_rn(e, p) > c) |
                              (y[0] != 0.0) | (y[1] != 0.0) | (y[2] != 0.0);
            bool any_th = false;
#ifdef MP_TIMELINE
            { const long long t = clock64(); c_ld += t - tq; tq = t; }
#endif
            if (need) {
                step3<UNIT>(p, c, e, wa, wc, we, y, k, viol, th);
                st_sh(pa[s], p);
                st_sh(pc[s], c);
                st_sh(pe[s], e);
                moved = true;
                any_th = (th[0] > THETA_FLOOR) | (th[1] > THETA_FLOOR) | (th[2] > THETA_FLOOR);
                // Cluster: x_ij and x_ik lie in this band's own rows (WR, or RK
                // rows i) and no later band (larger rows) reads those; x_jk is
                // read later by every later band if it is in WK (j > ihi), and
                // by the later bands up to the owner of row j if it is RK row j.
                if (fwd_band) fwd |= forward_jk(cc, (uint32_t)pe[s], e);
            }
#ifdef MP_TIMELINE
            { const long long t = clock64(); c_mt += t - tq; tq = t; }
#endif
            if (__any_sync(0xffffffffu, any_th))
                wr_append(dr, wd, cc->wp, cc->ctr, stream, bs, lane, th[0], th[1], th[2]);
#ifdef MP_TIMELINE
            { const long long t = clock64(); c_ap += t - tq; tq = t; }
#endif
        }
        if (__any_sync(0xffffffffu, moved) && Lc < Le) {
            unsigned f = 0;
#pragma unroll
            for (int u = 1; u < U; ++u) {
                const int Lx = Lc + u;
                if (Lx <= Le) {  // warp-uniform
                    int qa[S], qc[S], qe[S];
                    slot_addrs<S, W, ALIAS>(G, Lx, b, T.ihi, T.klo, qa, qc, qe);
#pragma unroll
                    for (int s = 0; s < S; ++s)
                        f |= triplet_violated(ld_sh(qa[s]), ld_sh(qc[s]), ld_sh(qe[s])) << (Lx - L0);
                }
            }
            todo = (todo & ((2u << (Lc - L0)) - 1u)) | __reduce_or_sync(0xffffffffu, f);
        }
        // next level to replay: flagged, or holding the next stored dual
        const unsigned rest = todo & ~((2u << (Lc - L0)) - 1u);
        int nxt = rest ? L0 + __ffs(rest) - 1 : Le + 1;
        if (dr.head < (uint32_t)(Le + 1 - T.Lbeg) * PER_LEVEL)
            nxt = min(nxt, T.Lbeg + (int)(dr.head / PER_LEVEL));
        Lc = nxt;
    }
#ifdef MP_TIMELINE
    if (cc->tl && lane == 0) {  // the caller's batch record, slots 3..7
        const int nb = wd->pad;  // batch index parked by the caller
        if (nb < TL_MAXB) {
            unsigned long long *r = cc->trace + (((size_t)band * 16 + warp) * TL_MAXB + nb) * TL_REC;
            // lookup, x loads + check, exact step + stores + forwarding, append
            r[4] = (unsigned long long)c_lk | ((unsigned long long)nlev << 48);
            // load+check | entries consumed << 32;  step | lookups, chunk switches << 32
            r[5] = (unsigned long long)c_ld | ((unsigned long long)(unsigned)wd->wpad[0] << 32);
            r[6] = (unsigned long long)c_mt | ((unsigned long long)(unsigned)wd->wpad[2] << 32);
            r[3] = 1ull | ((unsigned long long)(unsigned)wd->wpad[1] << 8);
            r[7] = (unsigned long long)c_ap | ((unsigned long long)(clock64() - tq0) << 32);
        }
    }
#endif
    // forwarded values land in the later bands before this warp's progress does
    if (__any_sync(0xffffffffu, fwd)) fence_cluster();
    return viol;
}

// ---------------------------------------------------------------------------
// warp-level dataflow
// ---------------------------------------------------------------------------
// Every conflict inside a tile is ordered along the (i,k) lattice: thread
// (i,k) may run level L once (i,k-1) and (i-1,k) have finished level L-1
// (this covers the aliased cross-role cases too: for any two conflicting
// triplets, the later one's (i,k) is reachable from the earlier one's by
// +1 steps in i or k, one level per step).  With the slot map
// q = warp*32*S + s*32 + lane (q = (i-ilo)*b + (k-klo), b <= 32*S), both
// neighbours of a warp's pairs live in the same warp or in warp-1, so a
// compute warp only waits for its predecessor's progress counter -- no CTA
// barrier per level, and a warp in the exact (cold) step delays only its
// successors.  A producer warp streams the j-rings: it lands blocks ahead of
// warp 0 and writes back blocks the last warp has passed.
__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];\n" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int *p, int v) {
    asm volatile("st.release.cta.shared.b32 [%0], %1;\n" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
// Progress store of a level that wrote nothing: the level's shared loads
// were consumed before this store issues, so no fence is needed for WAR.
__device__ __forceinline__ void st_relaxed(int *p, int v) {
    asm volatile("st.relaxed.cta.shared.b32 [%0], %1;\n" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
// spin until *p >= v (acquire), backing off so spinners do not steal issue slots
__device__ __forceinline__ void wait_geq(const int *p, int v, bool sleep) {
    if (ld_acquire(p) >= v) return;
    while (true) {
        if (sleep) __nanosleep(20);
        if (ld_acquire(p) >= v) return;
    }
}

struct alignas(16) TileSync {
    unsigned long long wkbar[32];  // per WK ring block slot: its TMA load landed
    int done[32];       // last level each compute warp finished
    int landed_by[16];  // highest ring block landed, per CTA of the cluster
    int lo_res;         // producer's lowest resident block (for the epilogue)
    int hi_issued;      // producer's highest issued block (for the epilogue)
    int pslow, pfast;   // producer-internal broadcast
    int blk0;           // the tile's first ring block (TMA slot phases count from it)
    int wb_lo;          // TMA producer: lowest block not yet written back (slots below are free)
    int wslow;          // TMA producer: writers' broadcast of the slowest warp's next level
    int df_hi;          // dataflow launch: highest ring block whose predecessors' data is visible
    int tile;           // dataflow launch: the tile this cluster claimed
};

// ---- dataflow launch: progress words in global memory --------------------
__device__ __forceinline__ int ld_acquire_gpu(const int32_t *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_relaxed_gpu(const int32_t *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Publish progress: the caller's (and, through the CTA barrier it passed,
// its peers') write-backs -- generic stores and completed bulk/TMA stores --
// happen before the release.
__device__ __forceinline__ void df_publish(int32_t *p, int v) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// After an acquire: later async-proxy (TMA / bulk) reads see the data.
__device__ __forceinline__ void df_after_acquire() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
// Highest ring block this tile may load given the predecessors' progress
// values r (row) and c (column): block g needs c > g; and, if it holds WR
// columns (16g < klo), r > g -- or the row predecessor finished once g
// reaches its RK columns [klo - b, klo) (g >= r_fin_blk = (klo - b) / 16;
// the later blocks of the prefix hold no WR column, so the prefix of
// loadable blocks ends at min(r, r_fin_blk) - 1 until the predecessor is done).
__device__ __forceinline__ int df_hi_of(const CtaConst *cc, int r, int c) {
    int hi = 0x3fffffff;
    if (cc->dep_c) hi = min(hi, c - 1);
    if (cc->dep_r && r < DF_DONE) hi = min(hi, min(r, cc->r_fin_blk) - 1);
    return hi;
}
// Poll the predecessors (relaxed) and return the highest loadable block;
// `seen` caches it; an advance is acquired (one acquire per advance).
__device__ __forceinline__ int df_poll(const CtaConst *cc, int &seen) {
    const int r = cc->dep_r ? ld_relaxed_gpu(cc->dep_r) : DF_DONE;
    const int c = cc->dep_c ? ld_relaxed_gpu(cc->dep_c) : DF_DONE;
    const int hi = df_hi_of(cc, r, c);
    if (hi > seen) {
        if (cc->dep_r) (void)ld_acquire_gpu(cc->dep_r);
        if (cc->dep_c) (void)ld_acquire_gpu(cc->dep_c);
        df_after_acquire();
        seen = hi;
    }
    return seen;
}
// Block until blocks up to g may be loaded.
__device__ __forceinline__ void df_wait_blk(const CtaConst *cc, int &seen, int g) {
    while (df_poll(cc, seen) < g) __nanosleep(64);
}

// Lowest ring block landed in every CTA of the cluster: a block may be used
// (and an upstream band may forward writes into it) only once every band's
// copy of it has landed.
// (Other bands' entries are back-pressure only -- this warp never reads their
// rings -- so relaxed loads do; the own band's ring data is acquired.)
// The other bands' entries are this CTA's own copies, stored remotely by
// their producers: a volatile shared load (LDS) sees them; a stale value only
// delays (entries grow monotonically), so no cluster-scope load is needed.
__device__ __forceinline__ int ld_volatile_sh(const int *p) {
    int v;
    asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
// Lowest landed block over the cluster's bands: the own band's entry with an
// acquire (this CTA's warps read that ring), the 16 entries with four vector
// loads issued together (entries past the cluster size hold 0x3fffffff) -- a
// loop of scalar volatile loads serialises and cost ~600 cycles per call on
// the tile's first warp (timeline build, every other ring block).
__device__ __forceinline__ int landed_min(TileSync &ts, int, int band) {
    int m = ld_acquire(&ts.landed_by[band]);
    const uint32_t a = smem_u32(&ts.landed_by[0]);
    int v[16];
#pragma unroll
    for (int q = 0; q < 4; ++q)
        asm volatile("ld.volatile.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v[4 * q]), "=r"(v[4 * q + 1]), "=r"(v[4 * q + 2]), "=r"(v[4 * q + 3])
                     : "r"(a + 16u * q)
                     : "memory");
#pragma unroll
    for (int q = 0; q < 16; ++q) m = min(m, v[q]);
    return m;
}

// Back-off of the progress spins: a sleeping warp frees issue slots but
// wakes late (measured: no difference between 0, 5, 20 and 100 ns).
#ifndef MP_SPIN_NS
#define MP_SPIN_NS 20
#endif
__device__ __forceinline__ void spin_pause() {
    if (MP_SPIN_NS > 0) __nanosleep(MP_SPIN_NS);
}

// spin until *p >= v (acquire); returns the value seen
__device__ __forceinline__ int wait_geq_v(const int *p, int v) {
    int x = ld_acquire(p);
    while (x < v) {
        spin_pause();
        x = ld_acquire(p);
    }
    return x;
}
// the same for a flag in another CTA of the cluster (shared::cluster
// address): poll with relaxed loads (a cluster-scope acquire is expensive),
// then one acquire of the value that satisfied the wait
__device__ __forceinline__ int wait_geq_cluster(uint32_t a, int v) {
    int x = ld_relaxed_cluster(a);
    while (x < v) {
        spin_pause();
        x = ld_relaxed_cluster(a);
    }
    // the relaxed load that saw x, then an acquire fence: synchronises with the
    // release that published x (a second, acquiring load would be another
    // ~600-cycle round trip through the cluster window)
    asm volatile("fence.acquire.sync_restrict::shared::cluster.cluster;" ::: "memory");
    return x;
}


// Sweep levels [La, Lb] of one phase.  Levels are taken in batches of U: in
// the common case nothing moves, so the U levels' checks read only data
// that is final (the predecessor warp is done with the batch's last level
// minus one) and can be issued together; progress is published once per
// batch.  If some level of the batch needs the exact step, the batch is
// finished level by level from that level on (later levels re-checked after
// the update).
template <int S, int W, bool UNIT, bool ALIAS, int U>
__device__ __forceinline__ void sweep(int La, int Lb, unsigned char *sm, const SlotGeom<S> &G,
                                      CtaConst &cc, TileSync &ts, WarpDuals *wd, DualRegs &dr, int warp,
                                      int b, int ihi, int klo, double &viol, int &nbatch) {
    if (La > Lb) return;
    constexpr uint32_t PER_LEVEL = (uint32_t)(S * 96);
    const TileDesc &T = cc.T;
    const int lane = threadIdx.x & 31;
    double xcr[S];
    // alias-free levels: x_ik is this thread's alone and lives in a register,
    // loaded once the first batch's dependencies are met (the previous
    // phase's last level may still write it in the predecessor warp)
#if defined(MP_TILETIME)
    const bool tr = cc.tt != nullptr;
#elif defined(MP_TRACE)
    const bool tr = cc.trace != nullptr;
#else
    constexpr bool tr = false;  // build with -DMP_TRACE for mp_trace counters
#endif
    unsigned long long c_pred = 0, c_ring = 0, c_hot = 0, c_cold = 0, c_rel = 0, n_cold = 0;
    long long t0 = tr ? clock64() : 0, t1;
    // Predecessors of this warp.  Row-major: the previous warp of the band,
    // and for warp 0 of a later band the previous band's last warp.
    // Column-major (cluster bands): the previous warp of the band (columns to
    // the left) and, in the previous band, the warp holding the last row of
    // this warp's rightmost column (so the warps form a 2-D grid: the chain
    // from the tile's first warp to its last is C + nwc long, not C*nwc).
    // A batch [L, Le] waits until each predecessor finished Le (- lead): by
    // induction every warp holding a lattice predecessor of this warp's slots
    // then reached Le - 1.  Remote flags are polled with cluster-scope
    // acquires; the values this warp needs from there were forwarded into its
    // own copies and fenced by their writers before those published progress.
    const int C = cc.C;
    const int lwS = cc.lw * S;
    const bool has_loc = warp > 0;
    const int *loc_flag = &ts.done[warp > 0 ? warp - 1 : 0];
    int rem_warp = cc.nwc - 1;
    if (cc.colm) {
        const int r0 = cc.bst[cc.band];
        const int rbc = max(1, min(min(b, (int)cc.bst[cc.band + 1]), T.ihi - T.ilo + 1) - r0);  // the band's real rows
        const int qmax = min(warp * lwS + lwS - 1, rbc * b - 1);
        const int kmax = max(qmax, 0) / rbc;
        if (cc.band > 0) {  // the previous band's slot of (its last row, column kmax)
            const int rp = cc.bst[cc.band] - cc.bst[cc.band - 1];
            rem_warp = min(cc.nwc - 1, (kmax * rp + rp - 1) / ((int)cc.blw[cc.band - 1] * S));
        }
    }
    const bool has_rem = cc.band > 0 && (cc.colm || warp == 0);
    const uint32_t rem_flag = has_rem ? mapa(smem_u32(&ts.done[rem_warp]), cc.band - 1) : 0u;
    // with whole tile rows per warp (lw*S >= b) and row-major slots every
    // neighbour is in this warp or the previous one: Le - 1 suffices (equal
    // to Le for aligned batches; it only matters at a phase's short batch)
    const int lead = (!cc.colm && lwS >= b) ? 1 : 0;
    int loc_seen = has_loc ? ld_acquire(loc_flag) : 0x3fffffff;
    int rem_seen = has_rem ? ld_acquire_cluster(rem_flag) : 0x3fffffff;
    int landed_seen = landed_min(ts, C, cc.band);
    const int jtop0 = T.ilo + klo;  // top j at level L is L - jtop0
    for (int L = La; L <= Lb;) {
        const int Le = min(L + U - 1, Lb);
        const uint32_t base0 = (uint32_t)(L - T.Lbeg) * PER_LEVEL;
#ifdef MP_TIMELINE
        const long long tl0 = clock64();
#endif
        // dependencies of the whole batch: predecessor done with Le-1; ring landed
#ifndef MP_EXP_NOWAIT
        if (loc_seen < Le - lead) loc_seen = wait_geq_v(loc_flag, Le - lead);
        if (rem_seen < Le) rem_seen = wait_geq_cluster(rem_flag, Le);
#endif
        if (tr) { t1 = clock64(); c_pred += t1 - t0; t0 = t1; }
        const int need = min(Le - jtop0, T.jhi) >> 4;
#ifdef MP_TIMELINE
        int tl_spins = 0;
#endif
#ifndef MP_EXP_NOWAIT
        while (landed_seen < need) {
            landed_seen = landed_min(ts, C, cc.band);
            if (landed_seen < need) spin_pause();
#ifdef MP_TIMELINE
            ++tl_spins;
#endif
        }
#endif
        if (tr) { t1 = clock64(); c_ring += t1 - t0; t0 = t1; }
#ifdef MP_TIMELINE
        const long long tl1 = clock64();
#endif
        if (!ALIAS && L == La) {
#pragma unroll
            for (int s = 0; s < S; ++s) xcr[s] = ld_sh(G.pik[s]);
        }
        // progress seen now, for the next batch
        const int lpf = has_loc ? ld_acquire(loc_flag) : 0x3fffffff;
        // (remote flags are read only when a wait needs them: a relaxed load per
        // batch issued here, to return under the batch's work, costs more than
        // it saves -- config 2 4.11 -> 4.22 ms/pass, config 3 81.9 -> 85.4)
        unsigned fl = 0;  // bit u: level L+u has a violated row in some slot of this lane
        if (Le - L + 1 == U) {
            // full batch: straight-line, so the U levels' loads overlap
#pragma unroll
            for (int u = 0; u < U; ++u) {
                int pa[S], pc[S], pe[S];
                fl |= (unsigned)level_hot<S, W, ALIAS>(sm, G, L + u, b, ihi, klo, pa, pc, pe, xcr) << u;
            }
        } else {
#pragma unroll 1
            for (int Lx = L; Lx <= Le; ++Lx) {
                int pa[S], pc[S], pe[S];
                fl |= (unsigned)level_hot<S, W, ALIAS>(sm, G, Lx, b, ihi, klo, pa, pc, pe, xcr) << (Lx - L);
            }
        }
        const unsigned wfl = __reduce_or_sync(0xffffffffu, fl);
        const uint32_t lim = base0 + (uint32_t)(Le - L + 1) * PER_LEVEL;
#ifndef MP_EXP_NOCOLD
        const bool go_cold = wfl != 0u || dr.head < lim;
#else
        const bool go_cold = false;  // timing experiment only: results are wrong
#endif
        if (tr) { t1 = clock64(); c_hot += t1 - t0; t0 = t1; n_cold += go_cold; }
        if (go_cold) {
            // first level that needs the exact step: flagged, or the next dual
            int first = wfl ? L + __ffs(wfl) - 1 : Le + 1;
            if (dr.head < lim) first = min(first, L + (int)((dr.head - base0) / PER_LEVEL));
#ifdef MP_TIMELINE
            if (lane == 0) wd->pad = nbatch;
            __syncwarp();
#endif
            if (S == 1) {
                viol = cold_batch<S, W, UNIT, ALIAS, U>(L, first, Le, wfl, &cc, wd, dr, warp, viol, G);
                if (!ALIAS) {  // the exact steps may have moved this thread's x_ik
#pragma unroll
                    for (int s = 0; s < S; ++s) xcr[s] = ld_sh(G.pik[s]);
                }
            } else {
                // level by level from `first`: skipped levels have no flag and
                // no dual; after a replayed level every later one is re-checked
                bool fwd = false, dirty = false;
                for (int Lc = first; Lc <= Le; ++Lc) {
                    const uint32_t bl = (uint32_t)(Lc - T.Lbeg) * PER_LEVEL;
                    if (!dirty && !((wfl >> (Lc - L)) & 1u) && !(dr.head < bl + PER_LEVEL)) continue;
                    dirty |= level_full<S, W, UNIT, ALIAS>(Lc, bl, sm, G, &cc, wd, dr, warp, b, ihi, klo, xcr,
                                                           viol, fwd);
                }
                if (__any_sync(0xffffffffu, fwd)) fence_cluster();
            }
        }
        if (tr) { t1 = clock64(); c_cold += t1 - t0; t0 = t1; }
        __syncwarp();
        if (lane == 0) {
            if (go_cold) st_release(&ts.done[warp], Le);  // publishes the exact steps' writes
            else st_relaxed(&ts.done[warp], Le);
        }
#ifdef MP_TIMELINE
        if (cc.tl && lane == 0 && nbatch < TL_MAXB) {
            unsigned long long *r = cc.trace + (((size_t)cc.band * 16 + warp) * TL_MAXB + nbatch) * TL_REC;
            r[0] = (unsigned long long)tl0;
            r[1] = (unsigned long long)tl1;
            r[2] = (unsigned long long)clock64();
            r[3] = go_cold ? (S == 1 ? r[3] : 1ull) : 0ull;  // cold_batch wrote 1 | chunk-wait cycles << 8
            // hot batches: ring polls of this batch and the blocks landed beyond the one needed
            if (!go_cold) r[3] = ((unsigned long long)tl_spins << 8) | ((unsigned long long)(landed_seen - need) << 32);
        }
#endif
        ++nbatch;
        loc_seen = max(loc_seen, lpf);
        L = Le + 1;
        if (tr) { t1 = clock64(); c_rel += t1 - t0; t0 = t1; }
    }
#ifdef MP_TILETIME
    if (tr && lane == 0) {
        atomicAdd(&cc.tt[4 + TR_PRED_WAIT], c_pred);
        atomicAdd(&cc.tt[4 + TR_RING_WAIT], c_ring);
        atomicAdd(&cc.tt[4 + TR_HOT], c_hot);
        atomicAdd(&cc.tt[4 + TR_COLD], c_cold);
        atomicAdd(&cc.tt[4 + TR_RELEASE], c_rel);
        atomicAdd(&cc.tt[4 + TR_LEVELS], (unsigned long long)(Lb - La + 1));
        atomicAdd(&cc.tt[4 + TR_COLD_CALLS], n_cold);
    }
    return;
#endif
    if (tr && lane == 0) {
        atomicAdd(&cc.trace[TR_PRED_WAIT], c_pred);
        atomicAdd(&cc.trace[TR_RING_WAIT], c_ring);
        atomicAdd(&cc.trace[TR_HOT], c_hot);
        atomicAdd(&cc.trace[TR_COLD], c_cold);
        atomicAdd(&cc.trace[TR_RELEASE], c_rel);
        atomicAdd(&cc.trace[TR_LEVELS], (unsigned long long)(Lb - La + 1));
        atomicAdd(&cc.trace[TR_COLD_CALLS], n_cold);
    }
}

// The producer warps (P of them, named barrier 1): keep the j-rings ahead
// of the fastest compute warp and write back what the slowest has passed.
// Ring slots of block g are reused by block g + W/BLK, which is loaded only
// after g was written back.
__device__ __forceinline__ void producer_bar(int nthreads) {
    asm volatile("bar.sync 1, %0;\n" ::"r"(nthreads) : "memory");
}

// WK ring block g (rows j in [16g, 16g+16), columns K) as one 2-D TMA box;
// slot barrier g % (W/BLK), phase ((g - blk0) / (W/BLK)) & 1 (blk0 = the
// tile's first block, so every slot starts at phase 0).
template <int W>
__device__ __forceinline__ void wk_tma_load(const CtaConst *cc, TileSync *ts, double *WK, int g) {
    unsigned long long *bar = &ts->wkbar[g & (W / BLK - 1)];
    mbar_expect_tx(bar, (unsigned)(cc->wkp * BLK * 8));  // the box is wkp columns wide
    tma_load_2d(smem_u32(WK + ((g * BLK) & (W - 1)) * cc->wkp), cc->tmap, cc->T.klo, g * BLK, bar);
}
template <int W>
__device__ __forceinline__ void wk_tma_wait(TileSync *ts, int g) {
    mbar_wait(&ts->wkbar[g & (W / BLK - 1)], (uint32_t)(((g - ts->blk0) / (W / BLK)) & 1));
}
// A WK block may be written back as a whole box when every row holds only
// this tile's x_jk (j > ihi, j >= jlo; rows j >= z hold only k <= j pairs,
// the unused lower triangle, written back unchanged) and K is b wide.
__device__ __forceinline__ bool wk_tma_store_ok(const CtaConst *cc, int g) {
    return cc->tmap != nullptr && cc->tma_st && cc->wkp == cc->b && g * BLK >= max(cc->T.jlo, cc->T.ihi + 1);
}
__device__ __forceinline__ void bulk_wait_read_all() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

template <int W, bool UNIT>
__device__ __noinline__ void ring_producer(unsigned char *sm, const CtaConst *cc, TileSync *ts,
                                           int nwc, int np, int lo_res, int hi_issued) {
    const TileDesc &T = cc->T;
    const int b = cc->b, lane = threadIdx.x & 31;
    const int ptid = threadIdx.x - nwc * 32, pn = np * 32;
    double *smd = reinterpret_cast<double *>(sm);
    const int C = cc->C, band = cc->band;
    const int r0 = cc->bst[band], r1 = min(b, (int)cc->bst[band + 1]);
    const bool last_band = band == C - 1;
    double *WR = smd, *WK = smd + SmemMap<W>{b, cc->RB, cc->wkp, cc->wrp}.wk() / 8;
    const int xsize = cc->xsize;
    const int blast = T.jhi / BLK;
    const uint32_t band0_done = C > 1 ? mapa(smem_u32(&ts->done[0]), 0) : 0u;
    const int nres = W / BLK;
    constexpr int LOOKAHEAD = MP_LOOKAHEAD;
    int landed = hi_issued;  // the prologue landed everything it issued
#ifdef MP_TIMELINE
    int nit = 0, nidle = 0;
    unsigned long long *tlr = (cc->tl && ptid == 0) ? cc->trace + ((size_t)band * 16 + nwc) * TL_MAXB * TL_REC : nullptr;
#endif
    while (true) {
#ifdef MP_TIMELINE
        const long long tp0 = clock64();
#endif
        // Progress of every compute warp, each read with acquire so their ring
        // writes up to that level are visible.  Later warps may run ahead of
        // earlier ones (done[w] <= done[w-1] + 1 bounds them only from above).
        if (ptid < 32) {
            int lv = lane < nwc ? ld_acquire(&ts->done[lane]) : 0x3fffffff;
            int slow = lv, fast = lane < nwc ? lv : -0x3fffffff;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                slow = min(slow, __shfl_xor_sync(0xffffffffu, slow, o));
                fast = max(fast, __shfl_xor_sync(0xffffffffu, fast, o));
            }
            if (lane == 0) {
                // load ahead of the cluster's fastest warp (band 0 leads)
                if (C > 1) fast = max(fast, ld_acquire_cluster(band0_done) + 2 * MP_BATCH);
                ts->pslow = slow + 1;  // next level of the slowest warp
                ts->pfast = fast + 1;  // next level of the fastest warp
                if (cc->my_prog) {     // dataflow launch: what the predecessors allow
                    int seen = ts->df_hi;
                    ts->df_hi = df_poll(cc, seen);
                }
            }
        }
        producer_bar(pn);
#ifdef MP_TIMELINE
        const long long tp1 = clock64();
#endif
        const int slow = ts->pslow, fast = ts->pfast;
        if (slow > T.Lend) break;
        bool busy = false, wk_elem = false;
        const int low_need = max(slow - T.ihi - T.z, T.jlo) / BLK;
        while (lo_res < low_need) {
            const bool st = last_band && wk_tma_store_ok(cc, lo_res);
            ring_block<W, false>(T, b, cc->wkp, cc->wrp, cc->ld, cc->x, WR, WK, lo_res, ptid, pn, r0, r1, last_band && !st);
            wk_elem |= last_band && !st;
            if (st && ptid == 0) {
                fence_proxy_async();  // the compute warps' (acquired) writes, to the async proxy
                tma_store_2d(cc->tmap, T.klo, lo_res * BLK, smem_u32(WK + ((lo_res * BLK) & (W - 1)) * cc->wkp));
            }
            ++lo_res;
            busy = true;
        }
        if (cc->my_prog && busy) {  // dataflow launch: publish the written-back blocks
            if (ptid == 0) bulk_wait_all();
            __threadfence_block();
            producer_bar(pn);
            if (ptid == 0) df_publish(cc->my_prog, lo_res);
        }
#ifdef MP_TIMELINE
        const long long tp2 = clock64();
#endif
        const int need_fast = min(fast - T.ilo - T.klo, T.jhi) / BLK;
        const int want = min(min(need_fast + LOOKAHEAD, blast), ts->df_hi);
        // A slot whose WK rows were just written back element by element (by
        // every producer thread, rows split over warps) may be refilled by the
        // loader thread's TMA box only after all of them have read it.
        if (wk_elem && cc->tmap && hi_issued < want && hi_issued + 1 - lo_res < nres) producer_bar(pn);
        while (hi_issued < want && hi_issued + 1 - lo_res < nres) {
            ++hi_issued;
            ring_block<W, true>(T, b, cc->wkp, cc->wrp, cc->ld, cc->x, WR, WK, hi_issued, ptid, pn, r0, r1, cc->tmap == nullptr);
            if (cc->tmap && ptid == 0) {
                bulk_wait_read_all();  // the slots' previous box store has read them
                fence_proxy_async();
                wk_tma_load<W>(cc, ts, WK, hi_issued);
            }
            if (!UNIT)
                ring_block<W, true>(T, b, cc->wkp, cc->wrp, cc->ld, const_cast<double *>(cc->winvx), WR + xsize,
                                    WK + xsize, hi_issued, ptid, pn, r0, r1, true);
            cp_async_commit();  // one group per block, same sequence in every thread
            busy = true;
        }
#ifdef MP_TIMELINE
        const long long tp3 = clock64();
        long long tp4 = tp3;
#endif
        if (landed < hi_issued) {
            // publish what has landed; only wait for the newest copies when the
            // fastest warp is about to need them
            int now;
            if (need_fast + 1 >= hi_issued - 1) {
                cp_async_wait_all();
                now = hi_issued;
            } else {
                cp_async_wait_2();
                now = hi_issued - 2;
            }
            if (cc->tmap)
                for (int g = landed + 1; g <= now; ++g) wk_tma_wait<W>(ts, g);
#ifdef MP_TIMELINE
            tp4 = clock64();
#endif
            if (now > landed) {
                __threadfence_block();
                producer_bar(pn);  // every producer thread's copies up to `now` landed
                // every CTA of the cluster learns this band's landed block: the
                // own CTA with a release (its warps read the ring), the others
                // relaxed (back-pressure for their forwarded writes only)
                if (ptid == band) st_release(&ts->landed_by[band], now);
                else if (ptid < C) st_relaxed_cluster(mapa(smem_u32(&ts->landed_by[band]), ptid), now);
                landed = now;
                busy = true;
            }
        }
#ifdef MP_TIMELINE
        if (!busy) ++nidle;
        if (tlr && busy && nit < TL_MAXB) {  // busy producer iteration (slot nwc of the band)
            unsigned long long *r = tlr + (size_t)nit * TL_REC;
            r[0] = (unsigned long long)tp0;
            r[1] = (unsigned long long)tp1;
            r[2] = (unsigned long long)tp2;
            r[3] = (unsigned long long)tp3;
            r[4] = (unsigned long long)tp4;
            r[5] = (unsigned long long)clock64();
            r[6] = ((unsigned long long)(unsigned)slow << 32) | (unsigned)fast;
            r[7] = ((unsigned long long)(unsigned)lo_res << 48) | ((unsigned long long)(unsigned)hi_issued << 32) |
                   ((unsigned long long)(unsigned)landed << 16) | (unsigned)min(nidle, 65535);
            ++nit;
        }
#endif
        if (!busy) __nanosleep(32);
        producer_bar(pn);  // ts->pslow/pfast may be rewritten next round
    }
    if (ptid == 0) {
        ts->lo_res = lo_res;
        ts->hi_issued = hi_issued;
        bulk_wait_all();  // box stores complete before the CTA exits
    }
}

// Producer for tiles whose WK moves as TMA boxes (W = I): one elected loader
// thread issues each block as one mbarrier transaction -- the WK box plus one
// 128-byte bulk row copy per WR row of the band -- and publishes landed
// blocks; two writer warps write back what the slowest compute warp passed.
// The two roles run decoupled (the loader's capacity check reads the
// writers' wb_lo), so a block's load never waits behind a write-back.
template <int W>
__device__ __noinline__ void ring_producer_tma(unsigned char *sm, const CtaConst *cc, TileSync *ts,
                                               int nwc, int lo_res, int hi_issued) {
    const TileDesc &T = cc->T;
    const int b = cc->b, lane = threadIdx.x & 31;
    const int ptid = threadIdx.x - nwc * 32;
    double *smd = reinterpret_cast<double *>(sm);
    const int C = cc->C, band = cc->band;
    const int r0 = cc->bst[band], r1 = min(b, (int)cc->bst[band + 1]);
    const bool last_band = band == C - 1;
    double *WR = smd, *WK = smd + SmemMap<W>{b, cc->RB, cc->wkp, cc->wrp}.wk() / 8;
    const int blast = T.jhi / BLK;
    constexpr int nres = W / BLK;
    if (ptid < 32) {
        if (lane != 0) return;
        // ---- loader --------------------------------------------------------
        const uint32_t band0_done = C > 1 ? mapa(smem_u32(&ts->done[0]), 0) : 0u;
        const int rows = max(0, min(r1, T.ihi - T.ilo + 1) - r0);  // band rows that exist
        const unsigned tx = (unsigned)(cc->wkp * BLK * 8 + rows * BLK * 8);
        int landed = hi_issued, published = hi_issued;
        int df_seen = ts->df_hi;  // dataflow launch: highest block the predecessors allow
        while (true) {
            int slow = 0x3fffffff, fast = -0x3fffffff;
            for (int w = 0; w < nwc; ++w) {
                const int v = ld_acquire(&ts->done[w]);
                slow = min(slow, v);
                fast = max(fast, v);
            }
            if (slow + 1 > T.Lend) break;
            // band 0 leads the cluster: load ahead of it (a hint, relaxed)
            if (C > 1) fast = max(fast, ld_relaxed_cluster(band0_done) + 2 * MP_BATCH);
            const int need_fast = min(fast + 1 - T.ilo - T.klo, T.jhi) / BLK;
            int want = min(need_fast + MP_LOOKAHEAD, blast);
            if (cc->my_prog && want > df_seen) want = min(want, df_poll(cc, df_seen));
            bool busy = false;
            if (hi_issued < want) {
                const int lo = ld_acquire(&ts->wb_lo);  // slots below lo were written back
                if (hi_issued < want && hi_issued + 1 - lo < nres) fence_proxy_async();
                while (hi_issued < want && hi_issued + 1 - lo < nres) {
                    const int g = ++hi_issued;
                    unsigned long long *bar = &ts->wkbar[g & (nres - 1)];
                    mbar_expect_tx(bar, tx);
                    tma_load_2d(smem_u32(WK + ((g * BLK) & (W - 1)) * cc->wkp), cc->tmap, T.klo, g * BLK, bar);
                    const uint32_t wslot = smem_u32(WR + ((g * BLK) & (W - 1)));
                    const double *src = cc->x + (int64_t)(T.ilo + r0) * cc->ld + g * BLK;
                    for (int ii = 0; ii < rows; ++ii)
                        bulk_g2s(wslot + (uint32_t)(ii * cc->wrp * 8), src + (int64_t)ii * cc->ld, BLK * 8, bar);
                    busy = true;
                }
            }
            // landed, in order; block only when the fastest warp needs the block next
            while (landed < hi_issued) {
                const int g = landed + 1;
                const uint32_t ph = (uint32_t)(((g - ts->blk0) / nres) & 1);
                if (!mbar_test(&ts->wkbar[g & (nres - 1)], ph)) {
                    if (need_fast + 1 < g) break;
                    mbar_wait(&ts->wkbar[g & (nres - 1)], ph);
                }
                landed = g;
            }
            if (landed > published) {
                // the own CTA with a release (its warps read the ring), the
                // others relaxed (back-pressure for their forwarded writes)
                st_release(&ts->landed_by[band], landed);
                for (int d = 0; d < C; ++d)
                    if (d != band) st_relaxed_cluster(mapa(smem_u32(&ts->landed_by[band]), (unsigned)d), landed);
                published = landed;
                busy = true;
            }
            if (!busy) __nanosleep(32);
        }
        for (int g = landed + 1; g <= hi_issued; ++g)  // the epilogue writes every issued block back
            mbar_wait(&ts->wkbar[g & (nres - 1)], (uint32_t)(((g - ts->blk0) / nres) & 1));
        ts->hi_issued = hi_issued;
        return;
    }
    // ---- writers (the other producer warps) ----------------------------------
    const int wtid = ptid - 32, wn = 32 * (int)(blockDim.x / 32 - nwc - 1);
    int lo = lo_res;
    while (true) {
        if (wtid < 32) {
            int v = wtid < nwc ? ld_acquire(&ts->done[wtid]) : 0x3fffffff;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
            if (wtid == 0) ts->wslow = v + 1;
        }
        asm volatile("bar.sync 2, %0;" ::"r"(wn) : "memory");
        const int slow = ts->wslow;
        if (slow > T.Lend) break;
        const int low_need = max(slow - T.ihi - T.z, T.jlo) / BLK;
        if (lo < low_need) {
            for (; lo < low_need; ++lo) {
                const bool st = last_band && wk_tma_store_ok(cc, lo);
                ring_block<W, false>(T, b, cc->wkp, cc->wrp, cc->ld, cc->x, WR, WK, lo, wtid, wn, r0, r1,
                                     last_band && !st);
                if (st && wtid == 0) {
                    fence_proxy_async();
                    tma_store_2d(cc->tmap, T.klo, lo * BLK, smem_u32(WK + ((lo * BLK) & (W - 1)) * cc->wkp));
                }
            }
            if (wtid == 0) {
                if (cc->my_prog) bulk_wait_all();  // dataflow: the box stores are complete in x
                else bulk_wait_read_all();         // the box stores have read their slots
            }
            asm volatile("bar.sync 2, %0;" ::"r"(wn) : "memory");
            if (wtid == 0) {
                st_release(&ts->wb_lo, lo);
                if (cc->my_prog) df_publish(cc->my_prog, lo);  // every writer's stores: the barrier above
            }
        } else {
            __nanosleep(64);
        }
        asm volatile("bar.sync 2, %0;" ::"r"(wn) : "memory");  // ts->wslow is rewritten next
    }
    if (wtid == 0) {
        ts->lo_res = lo;
        bulk_wait_all();  // box stores complete before the CTA exits
    }
}

// U = levels per batch (one progress publish per batch).  A warp trails its
// lattice predecessor by a batch, so the chain of warps from a tile's first
// to its last spans (warps in the chain) x U levels, which -- plus the 2b - 2
// levels of a warp's own j-window and the blocks loaded ahead -- must fit the
// ring or the first warps stall on ring slots the last ones still hold: the
// host picks U = 4 for the 2-CTA shape on the W = 256 ring and MP_BATCH = 8
// elsewhere (round_shape).
template <int S, int W, bool UNIT, int U = MP_BATCH>
__global__ void __launch_bounds__(MAX_CTA_THREADS, 1) tile_round_kernel(TileArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    __shared__ CtaConst cc;
    __shared__ TileSync ts;
    const long long tk0 = clock64();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nt = blockDim.x, nwc = a.nwc, np = nt / 32 - nwc;  // compute / producer warps
    // a cluster of C CTAs shares one tile: CTA `band` owns rows [r0, r1) (relative to ilo)
    const int C = (int)cluster_size();
    const int band = C > 1 ? (int)cluster_rank() : 0;
    // dataflow launch: the cluster claims the next tile of the launch's list
    // (in schedule order, so every tile it may wait on is claimed by a running
    // cluster); a per-round launch takes its tile from the grid position
    int tidx = (int)(blockIdx.x / C);
    if (a.df) {
        if (band == 0 && tid == 0) {
            const int t = atomicAdd(a.qctr, 1);
            for (int d = 0; d < C; ++d) st_relaxed_cluster(mapa(smem_u32(&ts.tile), (unsigned)d), t);
        }
        if (C > 1) cluster_sync_all();
        else __syncthreads();
        tidx = ts.tile;
        MP_ASSERT(tidx >= 0 && tidx < (int)(gridDim.x / C));
    }
    const TileDesc T = a.tiles[tidx];
    const int b = a.b;
    const int RB = a.rbmax;  // most rows of a band (the WR staging)
    const int r0 = a.bst[band], r1 = min(b, (int)a.bst[band + 1]);
    // Bands holding rows: all C, except for the first family's single-row
    // tiles (x = 1 - b: row 0 only), which run on band 0 alone -- the other
    // CTAs of the cluster only take part in its two barriers (no forwarding
    // to them, no lattice coupling; band 0 writes WK back).  The slot map of
    // a band covers its real rows (a single row's columns fill few warps).
    const int nrows = T.ihi - T.ilo + 1;
    int Ce = 0;
    for (int d = 0; d < C; ++d)
        if ((int)a.bst[d] < nrows) Ce = d + 1;
    const bool idle_band = band >= Ce;
    const bool last_band = band == Ce - 1;
    const int64_t stream_base = T.stream0 + (int64_t)band * nwc;
    const SmemMap<W> M{b, RB, a.wkp, a.wrp};
    // TMA boxes need a 16-byte aligned start column: tiles with an odd klo copy
    // WK element by element (the configs' even n give every tile an even klo)
    const void *tmap = (T.klo & 1) ? nullptr : a.tmap;
    // base aligned to W*8 bytes (the launch reserves the slack) so ring rows
    // are W*8-aligned shared addresses and a slot address is one LOP3
    unsigned char *sm = smem_raw + ((128 - (smem_u32(smem_raw) & 127)) & 127);
    const int B32 = (int)smem_u32(sm);
    double *smd = reinterpret_cast<double *>(sm);
    const int xb = M.xbytes();
    WarpDuals *wds = reinterpret_cast<WarpDuals *>(sm + xb * (UNIT ? 1 : 2));
    double *WR = smd + M.wr() / 8;
    double *WK = smd + M.wk() / 8;
    double *RK = smd + M.rk() / 8;
    const int xsize = xb / 8;  // doubles between x staging and winv staging
    if (tid == 0) {
        cc.T = T;
        cc.x = a.x;
        cc.winvx = a.winvx;
        cc.ld = a.ld;
        cc.eps = a.eps;
        cc.rp = a.rp;
        cc.wp = a.wp;
        cc.ctr = a.ctr;
        cc.b = b;
        cc.nt = nt;
        cc.xsize = xsize;
        cc.trace = a.trace;
        cc.kc = a.kc;
        cc.C = Ce;  // the cluster as far as the sweep is concerned (bands with rows)
        cc.band = band;
        cc.RB = RB;
        cc.nwc = nwc;
        cc.rep_lo = (uint32_t)B32 + (uint32_t)M.wk();
        cc.zero_lo = (uint32_t)B32 + (uint32_t)M.zero();
        cc.rk_lo = (uint32_t)B32 + (uint32_t)M.rk();
        cc.rk_row_mul = (uint32_t)((0x100000000ull + 8ull * (unsigned)b - 1) / (8ull * (unsigned)b));
        for (int d = 0; d <= C; ++d) cc.bst[d] = a.bst[d];
        for (int d = 0; d < C; ++d) cc.blw[d] = a.blw[d];
        for (int d = 0; d < C; ++d)
            for (int r = a.bst[d]; r < min(b, (int)a.bst[d + 1]) && r < 64; ++r) cc.rowband[r] = (uint8_t)d;
        cc.tmap = tmap;
        cc.tma_st = a.tma_store && T.z - T.klo + 1 == b;
        cc.wkp = a.wkp;
        cc.wrp = a.wrp;
        cc.tl = a.trace != nullptr && a.round_id == a.tl_round && tidx == a.tl_tile && band < 8;
        cc.B32 = B32;
        cc.lw = band_lanes(a.blw[band], nwc, S, max(1, min(r1, nrows) - r0), r1 - r0, b, a.colm != 0);
        cc.colm = a.colm;
        cc.tt = nullptr;
#ifdef MP_TILETIME
        {  // (a dataflow launch's tiles continue into the following round slots)
            const int rr = a.round_id + tidx / TT_TILES, tt = tidx % TT_TILES;
            if (a.trace && rr < TT_ROUNDS && band < TT_BANDS)
                cc.tt = a.trace + (((size_t)rr * TT_TILES + tt) * TT_BANDS + band) * TT_REC;
        }
#endif
        cc.dep_r = cc.dep_c = cc.dep_d = nullptr;
        cc.my_prog = nullptr;
        cc.r_fin_blk = 0;
        if (a.df) {
            const int4 dp = a.dep[tidx];
            MP_ASSERT(dp.x < tidx && dp.y < tidx && dp.z < tidx);  // claimed before this tile
            cc.my_prog = a.prog + (size_t)tidx * C + band;
            if (dp.x >= 0) cc.dep_r = a.prog + (size_t)dp.x * C + band;
            if (dp.y >= 0) cc.dep_c = a.prog + (size_t)dp.y * C + (C - 1);
            if (dp.z >= 0) cc.dep_d = a.prog + (size_t)dp.z * C;
            cc.r_fin_blk = max(T.klo - b, 0) / BLK;
        }
    }
    for (int e = tid; e < W; e += nt) smd[M.zero() / 8 + e] = 0.0;
    if (tid < 32) ts.done[tid] = T.Lbeg - 1;

    // Programmatic dependent launch: everything above reads only this launch's
    // arguments; x, the dual pools and the counters were written by the
    // previous round, so wait for it here.
    asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef MP_TILETIME
    __syncthreads();
    if (tid == 0 && cc.tt) {
        cc.tt[0] = gtimer();
        cc.tt[12] = (unsigned long long)(T.ilo + 1);  // 0 = no record
        cc.tt[13] = (unsigned long long)T.z;
        cc.tt[14] = (unsigned long long)C;
        cc.tt[15] = (unsigned long long)nwc;
    }
#endif

    // --- staging prologue (all threads) -----------------------------------
    const int blast = T.jhi / BLK;
    const int lo0 = max(T.Lbeg - T.ihi - T.z, T.jlo) / BLK;
    const int hi0 = min(min(T.Lbeg - T.ilo - T.klo, T.jhi) / BLK + 1, blast);
    ts.df_hi = 0x3fffffff;
    if (a.df) {  // the predecessors' write-backs this prologue reads
        if (tid == 0) {
            if (cc.dep_d) {  // near the diagonal: the diagonal predecessor finished (every band)
                for (int d = 0; d < C; ++d)
                    while (ld_relaxed_gpu(cc.dep_d + d) < DF_DONE) __nanosleep(64);
                for (int d = 0; d < C; ++d) (void)ld_acquire_gpu(cc.dep_d + d);
                df_after_acquire();
            }
            int seen = -1;
            df_wait_blk(&cc, seen, hi0);
            if (cc.dep_c) {  // RK rows [ilo, ihi]: the column predecessor's WK blocks up to ihi
                const int need = T.ihi / BLK + 1;
                while (ld_relaxed_gpu(cc.dep_c) < need) __nanosleep(64);
                (void)ld_acquire_gpu(cc.dep_c);
                df_after_acquire();
            }
            ts.df_hi = seen;
        }
        __syncthreads();
    }
    rk_block<true>(T, b, a.ld, a.x, RK, tid, nt, 0, b);
    if (!UNIT) rk_block<true>(T, b, a.ld, const_cast<double *>(a.winvx), RK + xsize, tid, nt, 0, b);
    if (tmap && tid == 0) {  // WK blocks by TMA (cc was written by this thread)
        ts.blk0 = lo0;
        ts.wb_lo = lo0;
        for (int s = 0; s < W / BLK; ++s) mbar_init(&ts.wkbar[s], 1);
        mbar_fence_init();
        for (int bk = lo0; bk <= hi0; ++bk) wk_tma_load<W>(&cc, &ts, WK, bk);
    }
    for (int bk = lo0; bk <= hi0; ++bk) {
        ring_block<W, true>(T, b, a.wkp, a.wrp, a.ld, a.x, WR, WK, bk, tid, nt, r0, r1, tmap == nullptr);
        if (!UNIT)
            ring_block<W, true>(T, b, a.wkp, a.wrp, a.ld, const_cast<double *>(a.winvx), WR + xsize, WK + xsize,
                                bk, tid, nt, r0, r1, true);
    }
    cp_async_commit();
    // every band lands the same prologue blocks; entries past the bands with
    // rows never move and must not bound landed_min
    if (tid < 16) ts.landed_by[tid] = tid < Ce ? hi0 : 0x3fffffff;
    WarpDuals *wd = wds + (warp < nwc ? warp : 0);
    DualRegs dr;
    if (warp < nwc) rd_init(dr, wd, a.rp, stream_base + warp, lane);
    cp_async_wait_all();
    if (tmap && tid == 0)
        for (int bk = lo0; bk <= hi0; ++bk) wk_tma_wait<W>(&ts, bk);
    __syncthreads();
    // no CTA may forward into (or publish to) a CTA before its staging landed
    if (C > 1) cluster_sync_all();
    const long long tk1 = clock64();
#ifdef MP_TILETIME
    if (tid == 0 && cc.tt) cc.tt[1] = gtimer();
#endif

    double viol = 0.0;
    if (idle_band) {  // no rows: nothing to sweep; the epilogue writes back nothing of it
        if (tid == 0) {
            ts.lo_res = lo0;
            ts.hi_issued = hi0;
        }
    } else if (warp >= nwc) {
        // (one CTA per tile: 40 WR rows per block are too many bulk copies for
        // one loader thread; the combined producer is faster there, config 5)
        if (UNIT && tmap && np >= 3 && C > 1 && !MP_OLD_PRODUCER)
            ring_producer_tma<W>(sm, &cc, &ts, nwc, lo0, hi0);
        else
            ring_producer<W, UNIT>(sm, &cc, &ts, nwc, np, lo0, hi0);
    } else {
        // --- per-slot geometry: q = warp*32*S + s*32 + lane -> (i,k) -------
        SlotGeom<S> G;
        slot_geom<S, W>(G, T, M, B32, b, r0, min(r1, nrows), warp, lane, cc.lw, a.colm != 0);
        const int ihi = T.ihi, klo = T.klo;
        // Level L touches j in [L-ihi-z, L-ilo-klo]: alias-free (no j in R or
        // K) iff L in (2*ihi + z, 2*klo + ilo).
        const int mid_a = max(2 * ihi + T.z + 1, T.Lbeg);
        const int mid_b = min(2 * klo + T.ilo - 1, T.Lend);
#ifdef MP_TIMELINE
        if (cc.tl && warp == 0 && lane == 0) {
            unsigned long long *r = cc.trace + (((size_t)band * 16 + 15) * TL_MAXB) * TL_REC;
            r[0] = (unsigned long long)clock64();
            r[1] = gtimer();
        }
#endif
        int nbatch = 0;
        if (mid_a <= mid_b) {
            sweep<S, W, UNIT, true, U>(T.Lbeg, mid_a - 1, sm, G, cc, ts, wd, dr, warp, b, ihi, klo, viol, nbatch);
            sweep<S, W, UNIT, false, U>(mid_a, mid_b, sm, G, cc, ts, wd, dr, warp, b, ihi, klo, viol, nbatch);
            sweep<S, W, UNIT, true, U>(mid_b + 1, T.Lend, sm, G, cc, ts, wd, dr, warp, b, ihi, klo, viol, nbatch);
        } else {
            sweep<S, W, UNIT, true, U>(T.Lbeg, T.Lend, sm, G, cc, ts, wd, dr, warp, b, ihi, klo, viol, nbatch);
        }
    }

    // --- epilogue: write back everything still staged ----------------------
    __syncthreads();
    // the next round may launch (its CTAs wait in griddepcontrol.wait until
    // this grid has finished and its writes are visible)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#ifdef MP_TIMELINE
    if (cc.tl && tid == 0) {
        unsigned long long *r = cc.trace + (((size_t)band * 16 + 15) * TL_MAXB) * TL_REC;
        r[2] = (unsigned long long)clock64();
        r[3] = gtimer();
        r[4] = (unsigned long long)tk0;
        r[5] = (unsigned long long)tk1;
    }
#endif
    const long long tk2 = clock64();
#ifdef MP_TILETIME
    if (tid == 0 && cc.tt) cc.tt[2] = gtimer();
#endif
    // own WR and RK rows (a row's final values live in its band); the last
    // band holds the final WK (every band forwards its WK writes downstream)
    for (int bk = ts.lo_res; bk <= ts.hi_issued; ++bk) {
        const bool st = last_band && wk_tma_store_ok(&cc, bk);
        ring_block<W, false>(T, b, a.wkp, a.wrp, a.ld, a.x, WR, WK, bk, tid, nt, r0, r1, last_band && !st);
        if (st && tid == 0) {  // wr_finish (warp 0) waits for the bulk group
            fence_proxy_async();
            tma_store_2d(tmap, T.klo, bk * BLK, smem_u32(WK + ((bk * BLK) & (W - 1)) * a.wkp));
        }
    }
    rk_block<false>(T, b, a.ld, a.x, RK, tid, nt, r0, r1);
    if (a.df) {  // this band's rows are final in x: successors may read them
        __syncthreads();
        if (tid == 0) {
            bulk_wait_all();  // this thread's box stores above
            df_publish(cc.my_prog, DF_DONE);
        }
    }
#ifdef MP_TRACE
    if (a.trace) {
        __syncthreads();
        if (tid == 0) {
            atomicAdd(&a.trace[TR_PROLOGUE], (unsigned long long)(tk1 - tk0));
            atomicAdd(&a.trace[TR_LOOP], (unsigned long long)(tk2 - tk1));
            atomicAdd(&a.trace[TR_EPILOGUE], (unsigned long long)(clock64() - tk2));
            atomicAdd(&a.trace[TR_EPI_BLOCKS], (unsigned long long)(ts.hi_issued - ts.lo_res + 1));
            atomicAdd(&a.trace[TR_CTAS], 1ull);
        }
    }
#endif
    if (warp < nwc) {
        wr_finish(dr, wd, a.wp, a.ctr, stream_base + warp, lane);
        viol = warp_max(viol);
        if (lane == 0) atomic_max_nonneg(&a.ctr->viol_bits, viol);
    }
    if (C > 1) cluster_sync_all();  // late remote stores must not hit an exited CTA
#ifdef MP_TILETIME
    if (tid == 0 && cc.tt) cc.tt[3] = gtimer();
#endif
}

// dynamic shared memory of one CTA
inline size_t tile_smem_bytes(int b, int W, bool unit, int nwc, int rb, int p, int pr) {
    const size_t xb = W == 512   ? SmemMap<512>{b, rb, p, pr}.xbytes()
                      : W == 256 ? SmemMap<256>{b, rb, p, pr}.xbytes()
                                 : SmemMap<128>{b, rb, p, pr}.xbytes();
    // 128 bytes of alignment slack; dual-stream state for the compute warps only
    return 128 + xb * (unit ? 1 : 2) + (size_t)nwc * sizeof(WarpDuals);
}

}  // namespace mp
