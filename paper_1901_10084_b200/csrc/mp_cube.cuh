// schedule_kind = "serial" as a cube wavefront.
//
// The reference's lexicographic sweep (_kernels.py:135-183, solver.py:125-
// 135) re-blocked: index blocks of CUBE_C, cubes (I, J, K), I <= J <= K, of
// triplets i < j < k with i in block I, j in J, k in K.  Two conflicting
// triplets share two indices and the later one (in lexicographic order) has
// the larger L = i+j+k, hence a block sum I+J+K no smaller; cubes with equal
// block sum share no pair.  So cube levels s = I+J+K in increasing order
// (one launch each, the level's cubes in any order -- one CTA per cube), and
// inside a cube the levels L in increasing order, reproduce the serial
// trajectory bit for bit (tests/test_schedule.py: test_cube_order_equals_serial).
// A pass is 3*ceil(n/CUBE_C) launches instead of 3n.
//
// A cube touches three CUBE_C x CUBE_C blocks of pairs -- (I,J), (I,K), (J,K),
// fewer when blocks coincide -- staged in shared memory for the whole cube;
// thread slot q = (warp*CUBE_S + s)*32 + lane owns (i, k) = (I*c + q/c,
// K*c + q%c) and at level L processes (i, L-i-k, k).  Levels are separated by
// a CTA barrier.  Hot/cold split and the dual streams (one per cube and warp,
// key = ((L - Lmin)*CUBE_S + s)*96 + lane*3 + kind) as in the tile kernel.
#pragma once

#include "mp_device.cuh"

namespace mp {

constexpr int CUBE_C = 32;      // cube edge
constexpr int CUBE_WARPS = 8;   // warps per CTA
constexpr int CUBE_S = CUBE_C * CUBE_C / (32 * CUBE_WARPS);  // slots per thread (4)

struct CubeDesc {
    int32_t I, J, K, pad;
    int64_t stream0;  // first warp stream of the cube
};

struct CubeArgs {
    double *x;            // dense n x ld
    const double *winvx;  // dense, general W only
    int64_t ld;
    int32_t n;
    const CubeDesc *cubes;  // this cube level's cubes
    DualPool rp, wp;
    PassCounters *ctr;
    StepConsts kc;
};

// shared-memory bytes of one cube CTA
inline size_t cube_smem_bytes(bool unit) {
    return (size_t)(unit ? 3 : 6) * CUBE_C * CUBE_C * 8 + 64 + CUBE_WARPS * sizeof(WarpDuals) + 128;
}

template <bool UNIT>
__global__ void __launch_bounds__(CUBE_WARPS * 32, 2) cube_level_kernel(CubeArgs a) {
    constexpr int c = CUBE_C, S = CUBE_S, cc2 = CUBE_C * CUBE_C;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nt = blockDim.x;
    const CubeDesc cd = a.cubes[blockIdx.x];
    const int I = cd.I, J = cd.J, K = cd.K, n = a.n;
    const int Ic = I * c, Jc = J * c, Kc = K * c;
    // distinct pair blocks: (I,J) -> 0, (I,K) -> s_ik, (J,K) -> s_jk
    const int s_ik = K == J ? 0 : 1;
    const int s_jk = I == J ? s_ik : (K == J ? 1 : 2);
    const int nblk = max(s_ik, s_jk) + 1;
    // x blocks [3][c*c], then (general W) their 1/reg_x mirror, a zero row
    // for inactive slots, the warps' dual-stream state
    double *blk = reinterpret_cast<double *>(smem_raw);
    double *zero = blk + (UNIT ? 3 : 6) * cc2;
    WarpDuals *wds = reinterpret_cast<WarpDuals *>(smem_raw + (UNIT ? 3 : 6) * cc2 * 8 + 64);
    const uint32_t B32 = smem_u32(blk);
    auto blk_rows = [&](int t, int &A, int &B) {  // block pair of staging slot t
        A = t == 0 || t == s_ik ? I : J;
        B = t == 0 ? J : K;
    };
    // stage the blocks (and 1/reg_x for general W)
    for (int t = 0; t < nblk; ++t) {
        int A, B;
        blk_rows(t, A, B);
        for (int e = tid; e < cc2; e += nt) {
            const int ar = A * c + e / c, bc = B * c + e % c;
            if (ar < bc && bc < n) {
                cp_async8(blk + t * cc2 + e, a.x + (int64_t)ar * a.ld + bc);
                if (!UNIT) cp_async8(blk + 3 * cc2 + t * cc2 + e, a.winvx + (int64_t)ar * a.ld + bc);
            }
        }
    }
    cp_async_commit();
    if (tid < 8) zero[tid] = 0.0;
    WarpDuals *wd = wds + warp;
    DualRegs dr;
    rd_init(dr, wd, a.rp, cd.stream0 + warp, lane);
    cp_async_wait_all();
    __syncthreads();

    // slot geometry
    int io[S], ko[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int q = (warp * S + s) * 32 + lane;
        io[s] = q / c;
        ko[s] = q % c;
    }
    const uint32_t zaddr = smem_u32(zero);
    const int xb = 3 * cc2 * 8;  // winv mirror offset (bytes)
    const int Lmin = Ic + Jc + Kc, Lmax = Lmin + 3 * c - 3;
    const StepConsts k = a.kc;
    const int64_t stream = cd.stream0 + warp;
    double viol = 0.0;
    for (int L = Lmin; L <= Lmax; ++L) {
        uint32_t pa[S], pc[S], pe[S];
        bool bad[S];
        bool any_bad = false;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int i = Ic + io[s], kk = Kc + ko[s], j = L - i - kk;
            const bool ok = j >= Jc && j < Jc + c && i < j && j < kk && kk < n;
            pa[s] = ok ? B32 + 8u * (uint32_t)(0 * cc2 + io[s] * c + (j - Jc)) : zaddr;
            pc[s] = ok ? B32 + 8u * (uint32_t)(s_ik * cc2 + io[s] * c + ko[s]) : zaddr;
            pe[s] = ok ? B32 + 8u * (uint32_t)(s_jk * cc2 + (j - Jc) * c + ko[s]) : zaddr;
            const double xa = ld_sh(pa[s]), xc = ld_sh(pc[s]), xe = ld_sh(pe[s]);
            bad[s] = (fabs(__dsub_rn(xa, xc)) > xe) | (__dsub_rn(xe, xa) > xc);
            any_bad |= bad[s];
        }
        const uint32_t base = (uint32_t)(L - Lmin) * (uint32_t)(S * 96);
        if (__any_sync(0xffffffffu, any_bad) || dr.head < base + (uint32_t)(S * 96)) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const uint32_t bs = base + (uint32_t)(s * 96);
                if (!(__any_sync(0xffffffffu, bad[s]) || dr.head < bs + 96u)) continue;
                double p = ld_sh(pa[s]), cx = ld_sh(pc[s]), e = ld_sh(pe[s]);
                double y[3] = {0.0, 0.0, 0.0};
                if (dr.head < bs + 96u) rd_lookup1(dr, wd, a.rp, bs, lane, y);
                double th[3] = {0.0, 0.0, 0.0};
                if (bad[s] | (y[0] != 0.0) | (y[1] != 0.0) | (y[2] != 0.0)) {
                    double wa = 1.0, wc = 1.0, we = 1.0;
                    if (!UNIT) {
                        wa = ld_sh(pa[s] + xb);
                        wc = ld_sh(pc[s] + xb);
                        we = ld_sh(pe[s] + xb);
                    }
                    step3<UNIT>(p, cx, e, wa, wc, we, y, k, viol, th);
                    st_sh(pa[s], p);
                    st_sh(pc[s], cx);
                    st_sh(pe[s], e);
                }
                if (__any_sync(0xffffffffu, (th[0] > THETA_FLOOR) | (th[1] > THETA_FLOOR) | (th[2] > THETA_FLOOR)))
                    wr_append(dr, wd, a.wp, a.ctr, stream, bs, lane, th[0], th[1], th[2]);
            }
        }
        __syncthreads();  // the next level reads this level's writes
    }
    // write back
    for (int t = 0; t < nblk; ++t) {
        int A, B;
        blk_rows(t, A, B);
        for (int e = tid; e < cc2; e += nt) {
            const int ar = A * c + e / c, bc = B * c + e % c;
            if (ar < bc && bc < n) a.x[(int64_t)ar * a.ld + bc] = blk[t * cc2 + e];
        }
    }
    wr_finish(dr, wd, a.wp, a.ctr, stream, lane);
    viol = warp_max(viol);
    if (lane == 0) atomic_max_nonneg(&a.ctr->viol_bits, viol);
}

}  // namespace mp
