// schedule_kind = "serial": the reference's lexicographic sweep
// (_kernels.py:135-183, solver.py:125-135) on the device.
//
// In lexicographic (i, j, k) order two conflicting triplets (sharing two
// indices) are always visited in increasing L = i+j+k, so
// a sweep over the levels L = 3 .. 3n-6, any order inside a level, gives the
// reference trajectory bit for bit.  One launch per level; inside a level a
// warp owns a row i and its lanes walk k (j = L-i-k), so x_ik and x_ij loads
// are row-contiguous.  x stays in the dense matrix in global memory (L2).
//
// Duals: one warp stream per (level, row i), key = (k - k_lo(L,i))*3 + kind,
// increasing in processing order; same chunk-record pool as the tiled path.
#pragma once

#include "mp_device.cuh"

namespace mp {

struct SerialArgs {
    double *x;             // dense n x ld
    const double *winvx;   // dense, general W only
    int64_t ld;
    int32_t n;
    double eps;
    DualPool rp, wp;
    PassCounters *ctr;
    StepConsts kc;
};

// k range of row i at level L: i < j = L-i-k < k <= n-1
__device__ __host__ __forceinline__ void serial_krange(int n, int L, int i, int &klo, int &khi) {
    klo = max(i + 2, (L - i) / 2 + 1);
    khi = min(n - 1, L - 2 * i - 1);
}

__host__ __device__ __forceinline__ int64_t serial_stream(int n, int L, int i) {
    return (int64_t)L * n + i;
}

template <bool UNIT>
__global__ void __launch_bounds__(256) serial_level_kernel(SerialArgs a, int L) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int n = a.n;
    const StepConsts sk = a.kc;
    double viol = 0.0;
    for (int i = gw; 3 * i + 3 <= L && i <= n - 3; i += nw) {
        int klo, khi;
        serial_krange(n, L, i, klo, khi);
        if (klo > khi) continue;
        const int64_t stream = serial_stream(n, L, i);
        // reader: this lane's entry of the current chunk
        int32_t rc = a.rp.head[stream];
        uint32_t rkey = KEY_END;
        double rval = 0.0;
        int rpos = 0;
        if (rc >= 0) {
            rkey = a.rp.rec[rc].keys[lane];
            rval = a.rp.rec[rc].vals[lane];
        }
        // writer state
        int32_t wc = -1, wfill = CHUNK;
        uint32_t wcount = 0;
        const double *xi = a.x + (int64_t)i * a.ld;
        for (int kc = klo; kc <= khi; kc += 32) {
            const int k = kc + lane;
            const bool act = k <= khi;
            const int j = L - i - k;
            const uint32_t base = (uint32_t)(kc - klo) * 3u;
            const uint32_t lim = base + 96u;
            // stored duals of this 32-wide chunk of k
            double y0 = 0.0, y1 = 0.0, y2 = 0.0;
            while (true) {
                const unsigned m = __ballot_sync(0xffffffffu, lane >= rpos && rkey < lim);
                unsigned mm = m;
                while (mm) {
                    const int src = __ffs(mm) - 1;
                    mm &= mm - 1;
                    const uint32_t key = __shfl_sync(0xffffffffu, rkey, src);
                    const double v = __shfl_sync(0xffffffffu, rval, src);
                    const uint32_t off = key - base;
                    if (off / 3u == (uint32_t)lane) {
                        const uint32_t kd = off % 3u;
                        if (kd == 0) y0 = v;
                        else if (kd == 1) y1 = v;
                        else y2 = v;
                    }
                }
                rpos += __popc(m);
                if (rpos < CHUNK || rc < 0) break;
                rc = a.rp.rec[rc].next;  // chunk exhausted: move on
                rpos = 0;
                rkey = KEY_END;
                if (rc >= 0) {
                    rkey = a.rp.rec[rc].keys[lane];
                    rval = a.rp.rec[rc].vals[lane];
                }
            }
            double t0 = 0.0, t1 = 0.0, t2 = 0.0;
            if (act) {
                double *pij = a.x + (int64_t)i * a.ld + j;
                double *pik = a.x + (int64_t)i * a.ld + k;
                double *pjk = a.x + (int64_t)j * a.ld + k;
                double p = *pij, c = xi[k], e = *pjk;
                const double d0 = __dsub_rn(__dsub_rn(p, c), e);
                const double d1 = __dsub_rn(__dsub_rn(c, p), e);
                const double d2 = __dsub_rn(__dsub_rn(e, p), c);
                if ((d0 > 0.0) | (d1 > 0.0) | (d2 > 0.0) | (y0 != 0.0) | (y1 != 0.0) |
                    (y2 != 0.0)) {
                    double wa = 1.0, wcc = 1.0, we = 1.0;
                    if (!UNIT) {
                        wa = a.winvx[(int64_t)i * a.ld + j];
                        wcc = a.winvx[(int64_t)i * a.ld + k];
                        we = a.winvx[(int64_t)j * a.ld + k];
                    }
                    t0 = dykstra_row<UNIT>(p, c, e, wa, wcc, we, y0, sk, viol);
                    t1 = dykstra_row<UNIT>(c, p, e, wcc, wa, we, y1, sk, viol);
                    t2 = dykstra_row<UNIT>(e, p, c, we, wa, wcc, y2, sk, viol);
                    *pij = p;
                    *pik = c;
                    *pjk = e;
                }
            }
            // append this chunk's thetas in (k, kind) order
            const bool h0 = t0 > THETA_FLOOR, h1 = t1 > THETA_FLOOR, h2 = t2 > THETA_FLOOR;
            const unsigned m0 = __ballot_sync(0xffffffffu, h0);
            const unsigned m1 = __ballot_sync(0xffffffffu, h1);
            const unsigned m2 = __ballot_sync(0xffffffffu, h2);
            if ((m0 | m1 | m2) && wc != -2) {
                const unsigned lt = (1u << lane) - 1u;
                const int before = __popc(m0 & lt) + __popc(m1 & lt) + __popc(m2 & lt);
                const int total = __popc(m0) + __popc(m1) + __popc(m2);
                const int nnew = (wfill + total + CHUNK - 1) / CHUNK - 1;
                int32_t c0 = 0;
                bool dead = false;
                if (nnew > 0) {
                    if (lane == 0) {
                        c0 = atomicAdd(&a.ctr->chunks_used, nnew);
                        if (c0 + nnew > a.wp.cap) {
                            atomicExch(&a.ctr->overflow, 1);
                            c0 = -1;
                        }
                    }
                    c0 = __shfl_sync(0xffffffffu, c0, 0);
                    dead = c0 < 0;
                    if (!dead) {
                        if (lane == 0) {
                            if (wc >= 0) a.wp.rec[wc].next = c0;
                            else a.wp.head[stream] = c0;
                        }
                        if (lane < nnew - 1) a.wp.rec[c0 + lane].next = c0 + lane + 1;
                    }
                }
                if (dead) {
                    wc = -2;
                } else {
                    int e = wfill + before;
                    const double th[3] = {t0, t1, t2};
                    const bool hk[3] = {h0, h1, h2};
#pragma unroll
                    for (int kd = 0; kd < 3; ++kd) {
                        if (hk[kd]) {
                            const int blk = e / CHUNK;
                            const int32_t c = blk == 0 ? wc : c0 + blk - 1;
                            a.wp.rec[c].keys[e - blk * CHUNK] = base + 3u * (uint32_t)lane + (uint32_t)kd;
                            a.wp.rec[c].vals[e - blk * CHUNK] = th[kd];
                            ++e;
                        }
                    }
                    if (nnew > 0) wc = c0 + nnew - 1;
                    wfill = wfill + total - CHUNK * nnew;
                    wcount += (uint32_t)total;
                }
            }
        }
        if (wc >= 0) {
            if (lane >= wfill) a.wp.rec[wc].keys[lane] = KEY_END;
            if (lane == 0) a.wp.rec[wc].next = -1;
        } else if (wc == -1 && lane == 0) {
            a.wp.head[stream] = -1;
        }
        if (lane == 0 && wcount) atomicAdd(&a.ctr->nnz, (unsigned long long)wcount);
    }
    viol = warp_max(viol);
    if (lane == 0) atomic_max_nonneg(&a.ctr->viol_bits, viol);
}

}  // namespace mp
