// Device kernels around the metric sweep: the pair phase fused with the
// per-pass objective / finiteness reductions, the exact violation scan, and
// packed <-> dense layout conversion.
#pragma once

#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

#include "mp_device.cuh"

namespace mp {

// Row start of pair (i, i+1) in the packed order (core.py:40-44).
__device__ __host__ __forceinline__ int64_t row_start(int64_t n, int64_t i) {
    return i * (n - 1) - i * (i - 1) / 2;
}

// Packed position p -> (i, j), i < j.
__device__ __forceinline__ void unpack_pair(int64_t p, int64_t n, int64_t &i, int64_t &j) {
    const double c = 2.0 * (double)n - 1.0;
    const double disc = c * c - 8.0 * (double)p;
    int64_t ii = (int64_t)floor((c - sqrt(disc > 0.0 ? disc : 0.0)) * 0.5);
    if (ii < 0) ii = 0;
    if (ii > n - 2) ii = n - 2;
    while (ii > 0 && row_start(n, ii) > p) --ii;
    while (ii < n - 2 && row_start(n, ii + 1) <= p) ++ii;
    i = ii;
    j = p - row_start(n, ii) + ii + 1;
}

// Block-wide sum of NV doubles in a fixed order; result valid in thread 0.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double *scratch /* [32*NV] */) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int c = 0; c < NV; ++c)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[c] += __shfl_down_sync(0xffffffffu, v[c], o);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int c = 0; c < NV; ++c) scratch[warp * NV + c] = v[c];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int c = 0; c < NV; ++c) v[c] = lane < nw ? scratch[lane * NV + c] : 0.0;
#pragma unroll
        for (int c = 0; c < NV; ++c)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v[c] += __shfl_down_sync(0xffffffffu, v[c], o);
    }
}

struct PairArgs {
    double *x;  // dense
    int64_t ld;
    double *f;                 // packed
    const double *d;           // packed
    const double *w;           // packed pair weights
    const double *winvx;       // dense (general W)
    const double *winvf;       // packed (general W)
    const double *regx;        // packed (general W)
    const double *regf;        // packed (general W)
    double *pu, *pl;           // packed pair duals (upper, lower)
    int64_t n, m;
    double eps;
    double *partials;  // [gridDim.x][4]: w.f, (rx x).x, (rf f).f, d.(pu-pl)
    PassCounters *ctr;
};

// Pair phase (_kernels.py:186-220) for every pair, fused with the sums of
// primal_objective (core.py:275-282) and b_dot_y (core.py:314-317) and the
// non-finite check of run_pass (solver.py:200-201).  Pair rows touch
// disjoint variables, so one thread per pair is exact.
template <bool UX, bool UF>
__global__ void __launch_bounds__(256) pair_phase_kernel(PairArgs a) {
    __shared__ double scratch[32 * 4];
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    double viol = 0.0;
    int bad = 0;
    const double eps = a.eps;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < a.m;
         p += (int64_t)gridDim.x * blockDim.x) {
        int64_t i, j;
        unpack_pair(p, a.n, i, j);
        const int64_t xo = i * a.ld + j;
        double x = a.x[xo], f = a.f[p];
        const double d = a.d[p];
        const double wx = UX ? 1.0 : a.winvx[xo];
        const double wf = UF ? 1.0 : a.winvf[p];
        const double s = __dadd_rn(wx, wf);
        // upper: x_ij - f_ij <= d_ij
        double y = a.pu[p];
        double d0 = __dsub_rn(__dsub_rn(x, f), d);
        viol = d0 > viol ? d0 : viol;
        double delta = __dadd_rn(d0, __ddiv_rn(__dmul_rn(y, s), eps));
        double theta = delta > 0.0 ? __ddiv_rn(__dmul_rn(eps, delta), s) : 0.0;
        double coef = __ddiv_rn(__dsub_rn(y, theta), eps);
        if (coef != 0.0) {
            x = __dadd_rn(x, UX ? coef : __dmul_rn(coef, wx));
            f = __dsub_rn(f, UF ? coef : __dmul_rn(coef, wf));
        }
        const double pu = theta > THETA_FLOOR ? theta : 0.0;
        // lower: -x_ij - f_ij <= -d_ij
        y = a.pl[p];
        d0 = __dsub_rn(__dsub_rn(d, x), f);
        viol = d0 > viol ? d0 : viol;
        delta = __dadd_rn(d0, __ddiv_rn(__dmul_rn(y, s), eps));
        theta = delta > 0.0 ? __ddiv_rn(__dmul_rn(eps, delta), s) : 0.0;
        coef = __ddiv_rn(__dsub_rn(y, theta), eps);
        if (coef != 0.0) {
            x = __dsub_rn(x, UX ? coef : __dmul_rn(coef, wx));
            f = __dsub_rn(f, UF ? coef : __dmul_rn(coef, wf));
        }
        const double pl = theta > THETA_FLOOR ? theta : 0.0;
        a.x[xo] = x;
        a.f[p] = f;
        a.pu[p] = pu;
        a.pl[p] = pl;
        // objective pieces on the post-pass state
        acc[0] += a.w[p] * f;
        acc[1] += (UX ? x : a.regx[p] * x) * x;
        acc[2] += (UF ? f : a.regf[p] * f) * f;
        acc[3] += d * (pu - pl);
        bad |= !(isfinite(x) && isfinite(f));
    }
    viol = warp_max(viol);
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(&a.ctr->viol_bits, viol);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicExch(&a.ctr->nonfinite, 1);
    block_sum<4>(acc, scratch);
    if (threadIdx.x == 0)
        for (int c = 0; c < 4; ++c) a.partials[blockIdx.x * 4 + c] = acc[c];
}

struct DevStats {
    double primal, dual, gap, viol;
    unsigned long long nnz;
    int32_t chunks_used, overflow, nonfinite, pad;
};

// Deterministic final reduction -> PassStats fields (run_pass,
// solver.py:202-210; objectives core.py:275-282, :330-339).
__global__ void __launch_bounds__(1024) finalize_kernel(const double *partials, int nparts,
                                                        double eps, const PassCounters *ctr,
                                                        DevStats *out) {
    __shared__ double scratch[32 * 4];
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int t = threadIdx.x; t < nparts; t += blockDim.x)
        for (int c = 0; c < 4; ++c) acc[c] += partials[t * 4 + c];
    block_sum<4>(acc, scratch);
    if (threadIdx.x == 0) {
        const double lin = acc[0], quad = acc[1] + acc[2], bdy = acc[3];
        const double primal = lin + 0.5 * eps * quad;
        const double dual = -bdy - 0.5 * eps * quad;
        out->primal = primal;
        out->dual = dual;
        out->gap = primal - dual;
        out->viol = __longlong_as_double((long long)ctr->viol_bits);
        out->nnz = ctr->nnz;
        out->chunks_used = ctr->chunks_used;
        out->overflow = ctr->overflow;
        out->nonfinite = ctr->nonfinite;
    }
}

// packed <-> dense (upper triangle) conversion
__global__ void expand_kernel(const double *packed, double *dense, int64_t ld, int64_t n, int64_t m) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
         p += (int64_t)gridDim.x * blockDim.x) {
        int64_t i, j;
        unpack_pair(p, n, i, j);
        dense[i * ld + j] = packed[p];
    }
}
__global__ void pack_kernel(const double *dense, double *packed, int64_t ld, int64_t n, int64_t m) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
         p += (int64_t)gridDim.x * blockDim.x) {
        int64_t i, j;
        unpack_pair(p, n, i, j);
        packed[p] = dense[i * ld + j];
    }
}

// Pair duals for export: (upper, lower) interleaved as the reference's
// (npairs, 2) array (core.py:224-228).
__global__ void interleave2_kernel(const double *a, const double *b, double *out, int64_t m) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
         p += (int64_t)gridDim.x * blockDim.x) {
        out[2 * p] = a[p];
        out[2 * p + 1] = b[p];
    }
}

// Exact violation scan (_kernels.py:28-57): every metric row of every
// triplet and both pair rows of every pair.  One CTA per smallest index i
// (heaviest rows first), warps over j, lanes over k -- x_ik and x_jk are
// row-contiguous in the dense layout, so every load is coalesced.
__global__ void __launch_bounds__(256) scan_metric_kernel(const double *x, int64_t ld, int64_t n,
                                                          unsigned long long *out) {
    const int64_t i = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double viol = 0.0;
    if (i < n - 2) {
        const double *xi = x + i * ld;
        for (int64_t j = i + 1 + warp; j < n - 1; j += nw) {
            const double xij = xi[j];
            const double *xj = x + j * ld;
            for (int64_t k = j + 1 + lane; k < n; k += 32) {
                const double xik = xi[k], xjk = xj[k];
                const double v1 = __dsub_rn(__dsub_rn(xij, xik), xjk);
                const double v2 = __dsub_rn(__dsub_rn(xik, xij), xjk);
                const double v3 = __dsub_rn(__dsub_rn(xjk, xij), xik);
                viol = v1 > viol ? v1 : viol;
                viol = v2 > viol ? v2 : viol;
                viol = v3 > viol ? v3 : viol;
            }
        }
    }
    viol = warp_max(viol);
    if (lane == 0) atomic_max_nonneg(out, viol);
}

__global__ void scan_pair_kernel(const double *x, int64_t ld, const double *f, const double *d,
                                 int64_t n, int64_t m, unsigned long long *out) {
    double viol = 0.0;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
         p += (int64_t)gridDim.x * blockDim.x) {
        int64_t i, j;
        unpack_pair(p, n, i, j);
        const double xv = x[i * ld + j];
        const double vu = __dsub_rn(__dsub_rn(xv, f[p]), d[p]);
        const double vl = __dsub_rn(__dsub_rn(d[p], xv), f[p]);
        viol = vu > viol ? vu : viol;
        viol = vl > viol ? vl : viol;
    }
    viol = warp_max(viol);
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out, viol);
}

// Dykstra start f = (-w) / (eps * reg_f) (solver.py:108-113), the reference's
// association and IEEE division (reg_f null: W = I, eps * 1.0 = eps exactly)
__global__ void f_init_kernel(const double *w, const double *regf, double eps, double *f, int64_t m) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
         p += (int64_t)gridDim.x * blockDim.x)
        f[p] = __ddiv_rn(-w[p], __dmul_rn(eps, regf ? regf[p] : 1.0));
}

__global__ void reciprocal_kernel(const double *in, double *out, int64_t m) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
         p += (int64_t)gridDim.x * blockDim.x)
        out[p] = __ddiv_rn(1.0, in[p]);
}

// ---------------------------------------------------------------------------
// g = c + A^T y from stored duals (core.accumulate_aty, core.py:285-293;
// SURVEY.md 8(f) rank 3).  The reference adds, per target position, the
// contributions of the stored duals in DualStore.items() order (metric keys in
// store order, three row entries each: core.py:296-311), then the pair duals
// (upper, then lower, core.py:244-253).  The device reproduces that order
// bit for bit: one record per metric row entry (record r = 3e + slot), a
// stable radix sort of the records by target keeps r ascending inside a
// target, and one thread per target segment adds sequentially from g = c.
// ---------------------------------------------------------------------------
// keys -> (target, record) pairs; slot 0 is the +1 entry, slots 1, 2 the -1s
__global__ void aty_records_kernel(const int64_t *keys, int64_t nnz, int64_t n, uint32_t *tgt,
                                   uint32_t *rec, int *bad) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t code = keys[e];
        const int64_t kind = code % 3, t3 = code / 3;
        const int64_t k = t3 % n, j = (t3 / n) % n, i = t3 / (n * n);
        if (code < 0 || !(i < j && j < k && k < n)) {
            atomicExch(bad, 1);
            tgt[3 * e] = tgt[3 * e + 1] = tgt[3 * e + 2] = 0;
        } else {
            const int64_t pij = row_start(n, i) + (j - i - 1);
            const int64_t pik = row_start(n, i) + (k - i - 1);
            const int64_t pjk = row_start(n, j) + (k - j - 1);
            // METRIC_IJ (pij, pik, pjk), METRIC_IK (pik, pij, pjk), METRIC_JK (pjk, pij, pik)
            tgt[3 * e] = (uint32_t)(kind == 0 ? pij : (kind == 1 ? pik : pjk));
            tgt[3 * e + 1] = (uint32_t)(kind == 0 ? pik : pij);
            tgt[3 * e + 2] = (uint32_t)(kind == 2 ? pik : pjk);
        }
        rec[3 * e] = (uint32_t)(3 * e);
        rec[3 * e + 1] = (uint32_t)(3 * e + 1);
        rec[3 * e + 2] = (uint32_t)(3 * e + 2);
    }
}

// g[0:m] = c[0:m] + metric contributions (sorted records), one thread per
// target segment, sequential in record order; coef * y is y or -y exactly
__global__ void aty_segments_kernel(const uint32_t *tgt, const uint32_t *rec, int64_t nrec,
                                    const double *vals, double *g) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nrec;
         t += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t p = tgt[t];
        if (t > 0 && tgt[t - 1] == p) continue;
        double acc = g[p];
        for (int64_t u = t; u < nrec && tgt[u] == p; ++u) {
            const uint32_t r = rec[u];
            const double y = vals[r / 3];
            acc = __dadd_rn(acc, (r % 3 == 0) ? y : -y);
        }
        g[p] = acc;
    }
}

// pair rows after every metric row (items() order): upper (p: +yu, m+p: -yu)
// then lower (p: -yl, m+p: -yl); zero duals are not stored, so not added
__global__ void aty_pairs_kernel(const double *pd, const double *c, double *g, int64_t m) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
         p += (int64_t)gridDim.x * blockDim.x) {
        const double yu = pd[2 * p], yl = pd[2 * p + 1];
        double gx = g[p], gf = c[m + p];
        if (yu != 0.0) {
            gx = __dadd_rn(gx, yu);
            gf = __dadd_rn(gf, -yu);
        }
        if (yl != 0.0) {
            gx = __dadd_rn(gx, -yl);
            gf = __dadd_rn(gf, -yl);
        }
        g[p] = gx;
        g[m + p] = gf;
    }
}

// ---------------------------------------------------------------------------
// correlation-clustering instance from a graph (instance.cc_instance,
// instance.py:124-161)
// ---------------------------------------------------------------------------
// Closed-neighbourhood intersections |N[a] & N[b]| for a < b: node u adds 1
// to every pair of N[u] = adj(u) + {u} (the sparse product B*B^T of the
// reference, instance.py:124-139, one warp per node).
__global__ void cc_inter_kernel(const int64_t *rowptr, const int32_t *cols, int64_t n,
                                uint32_t *inter) {
    const int lane = threadIdx.x & 31;
    const int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (u >= n) return;
    const int64_t r0 = rowptr[u], deg = rowptr[u + 1] - r0, sz = deg + 1;
    // element t of N[u]: the neighbours in order, then u itself
    for (int64_t t = 0; t < sz; ++t) {
        const int64_t a = t < deg ? cols[r0 + t] : u;
        for (int64_t q = lane; q < sz; q += 32) {
            const int64_t bq = q < deg ? cols[r0 + q] : u;
            if (a < bq) atomicAdd(&inter[row_start(n, a) + (bq - a - 1)], 1u);
        }
    }
}

// J = inter / union, s = log((1 + J - guard) / (1 - J + guard)) clipped to
// [-cap, cap] and pushed off zero by the offset; d = s < 0, w = |s|, packed
// pair order -- numpy's elementwise operations in the same order
// (instance.py:143-161).
__global__ void cc_map_kernel(const uint32_t *inter, const int64_t *rowptr, int64_t n, int64_t m,
                              double guard, double cap, double offset, double *d, double *w) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
         p += (int64_t)gridDim.x * blockDim.x) {
        int64_t i, j;
        unpack_pair(p, n, i, j);
        const double in = (double)inter[p];
        const double si = (double)(rowptr[i + 1] - rowptr[i] + 1);
        const double sj = (double)(rowptr[j + 1] - rowptr[j] + 1);
        const double un = __dsub_rn(__dadd_rn(si, sj), in);
        const double J = __ddiv_rn(in, un);
        const double num = __dsub_rn(__dadd_rn(1.0, J), guard);
        const double den = __dadd_rn(__dsub_rn(1.0, J), guard);
        double s = log(__ddiv_rn(num, den));
        s = fmin(fmax(s, -cap), cap);
        s = s >= 0.0 ? __dadd_rn(s, offset) : __dsub_rn(s, offset);
        d[p] = s < 0.0 ? 1.0 : 0.0;
        w[p] = fabs(s);
    }
}

// ---------------------------------------------------------------------------
// projection.dykstra_step (projection.py:63-87): single constraint rows applied
// in order by one thread, in that function's own association -- the sums over
// the row's entries start from 0 and b is subtracted last (for the lower pair
// row that is ((0 - x) - f) - (-d), not the sweep kernel's (d - x) - f), and
// W^-1 is formed as 1/reg per entry.
// ---------------------------------------------------------------------------
struct StepRow {
    int32_t nent, pad;   // 2 (pair row) or 3 (metric row)
    int64_t pos[3];      // positions in the value vector
    double coef[3];      // +-1 (core._row_entries)
    double reg[3];       // reg_x / reg_f of each entry
    double rhs;          // b of the row (0 metric, +d upper, -d lower)
    double y;            // old dual, >= 0
};

__global__ void single_steps_kernel(const StepRow *rows, int64_t nrows, double eps, double *v,
                                    double *theta_out, int32_t *changed_out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int64_t r = 0; r < nrows; ++r) {
        const StepRow R = rows[r];
        double winv[3], acc = 0.0, s = 0.0;
        for (int e = 0; e < R.nent; ++e) {
            winv[e] = __ddiv_rn(1.0, R.reg[e]);
            acc = __dadd_rn(acc, __dmul_rn(R.coef[e], v[R.pos[e]]));
        }
        const double d0 = __dsub_rn(acc, R.rhs);
        for (int e = 0; e < R.nent; ++e)
            s = __dadd_rn(s, __dmul_rn(__dmul_rn(R.coef[e], R.coef[e]), winv[e]));
        const double delta = __dadd_rn(d0, __ddiv_rn(__dmul_rn(R.y, s), eps));
        double theta = delta > 0.0 ? __ddiv_rn(__dmul_rn(eps, delta), s) : 0.0;
        const double coef = __ddiv_rn(__dsub_rn(R.y, theta), eps);
        if (coef != 0.0)
            for (int e = 0; e < R.nent; ++e)
                v[R.pos[e]] = __dadd_rn(v[R.pos[e]], __dmul_rn(__dmul_rn(coef, R.coef[e]), winv[e]));
        theta_out[r] = theta <= THETA_FLOOR ? 0.0 : theta;
        changed_out[r] = coef != 0.0;
    }
}

}  // namespace mp
