// Sharded execution of one instance over several GPUs.
//
// The tiles of a round are pairwise conflict-free (schedule.py:235-250), so
// a round's tiles are spread over the ranks (longest-processing-time per
// round, distributed.shard_rounds) and each tile always runs on the same rank,
// which therefore keeps its duals.  Every rank holds the whole
// x.  After each round a rank publishes the *footprint* of each of its tiles
// -- exactly the pairs the tile kernel writes back (ring_block / rk_block
// predicates in mp_device.cuh) -- and every rank applies the other ranks'
// footprints, so before round r+1 all ranks hold the x a single GPU would.
// Footprints of one round are disjoint, so the order of application does not
// matter and the result is bitwise the single-GPU trajectory.
//
// Footprint layout (padded, coalesced; `count` values per tile):
//   WR part  b rows i = ilo+ii      x wrw columns j = wr0 + c  (x_ij, j < klo)
//   RK part  b rows i = ilo+ii      x b   columns k = klo + kk (x_ik)
//   WK part  nwk rows j = wk0 + jj  x b   columns k = klo + kk (x_jk, j > ihi)
// Slots outside the tile's pairs (i >= j, k > z, ...) are padding: packed as
// garbage, never unpacked.
#pragma once

#include <cstdint>

#include "mp_device.cuh"

namespace mp {

struct FootDesc {
    TileDesc t;
    int64_t off;    // offset of this footprint in its owner's round buffer
    int32_t wr0;    // first WR column: max(jlo, ilo+1)
    int32_t wrw;    // WR row width: max(0, min(jhi, klo-1) - wr0 + 1)
    int32_t wk0;    // first WK row: max(jlo, ihi+1)
    int32_t nwk;    // WK rows: max(0, jhi - wk0 + 1)
    int32_t owner;  // rank that runs the tile
    int32_t pad;
};

__host__ __device__ inline int64_t foot_count(const FootDesc &f, int b) {
    return (int64_t)b * f.wrw + (int64_t)b * b + (int64_t)f.nwk * b;
}

// Element e of a footprint -> (row, col) and whether it is one of the tile's
// write-back pairs.
__device__ __forceinline__ bool foot_elem(const FootDesc &f, int b, int64_t e, int &row, int &col) {
    const TileDesc &T = f.t;
    const int64_t nwr = (int64_t)b * f.wrw;
    if (e < nwr) {
        const int ii = (int)(e / f.wrw);
        row = T.ilo + ii;
        col = f.wr0 + (int)(e - (int64_t)ii * f.wrw);
        return row <= T.ihi && col >= T.jlo && col <= T.jhi && col < T.klo && row < col;
    }
    e -= nwr;
    if (e < (int64_t)b * b) {
        const int ii = (int)(e / b);
        row = T.ilo + ii;
        col = T.klo + (int)(e - (int64_t)ii * b);
        return row <= T.ihi && col <= T.z && row < col;
    }
    e -= (int64_t)b * b;
    const int jj = (int)(e / b);
    row = f.wk0 + jj;
    col = T.klo + (int)(e - (int64_t)jj * b);
    return jj < f.nwk && col <= T.z && row < col;
}

// PACK: copy the footprints of `rank`'s tiles from x into buf (its round
// buffer).  !PACK: write the footprints of every other rank's tiles from
// buf + owner*stride into x.  One CTA per tile of the round.
template <bool PACK>
__global__ void __launch_bounds__(256) foot_copy_kernel(const FootDesc *fd, double *x, int64_t ld,
                                                        int b, double *buf, int64_t stride,
                                                        int rank) {
    const FootDesc f = fd[blockIdx.x];
    if (PACK ? f.owner != rank : f.owner == rank) return;
    double *base = buf + (PACK ? 0 : (int64_t)f.owner * stride) + f.off;
    const int64_t cnt = foot_count(f, b);
    for (int64_t e = threadIdx.x; e < cnt; e += blockDim.x) {
        int row, col;
        if (!foot_elem(f, b, e, row, col)) continue;
        double *gp = x + (int64_t)row * ld + col;
        if (PACK) base[e] = *gp;
        else *gp = base[e];
    }
}

// Local transport (several sessions of one process, test harness): the
// all-reduce of the per-pass counters over the group -- sum of nnz, max of
// the violation bits and the overflow flag -- written back to every member.
__global__ void reduce_counters_kernel(PassCounters *const *ctrs, int world) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    unsigned long long nnz = 0, viol = 0;
    int32_t ovf = 0;
    for (int g = 0; g < world; ++g) {
        nnz += ctrs[g]->nnz;
        viol = viol > ctrs[g]->viol_bits ? viol : ctrs[g]->viol_bits;
        ovf = ovf > ctrs[g]->overflow ? ovf : ctrs[g]->overflow;
    }
    for (int g = 0; g < world; ++g) {
        ctrs[g]->nnz = nnz;
        ctrs[g]->viol_bits = viol;
        ctrs[g]->overflow = ovf;
    }
}

}  // namespace mp
