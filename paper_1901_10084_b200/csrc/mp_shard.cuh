// Sharded execution of one instance over several GPUs.
//
// The tiles of a round are pairwise conflict-free (schedule.py:235-250), so
// a round's tiles are spread over the ranks (longest-processing-time per
// round, distributed.shard_rounds) and each tile always runs on the same rank,
// which therefore keeps its duals.  Every rank holds a whole
// x, but between the pair phases only the blocks a rank is about to touch are
// kept current: tiles and pairs live on one grid of b x b blocks (row block I
// = rows [1 + (I-1) b, I b], column block K = columns [n - b - K b, n - 1 -
// K b]), a tile's footprint -- exactly the pairs the tile kernel writes back
// (ring_block / rk_block predicates in mp_device.cuh) -- is a union of whole
// grid blocks, and the tiles touching one block form a fixed sequence in
// schedule order (distributed.block_touchers).  After each round a rank sends
// every block of its tiles' footprints to the rank of the block's *next
// toucher* only (distributed.next_toucher; nothing when that is the same
// rank), and a block's last toucher of the pass sends it to every rank, so
// all ranks enter the pair phase with the single-GPU x.  A tile thus reads
// exactly what a single GPU would have in x, and the trajectory is bitwise
// the single-GPU one.  Per rank that is ~(G-1)/G^2 of the touched pairs per
// pass instead of the (G-1)/G an all-gather of every footprint moves.
//
// A piece is a rectangle of x (rows [row0, row0 + nrows) x columns [col0,
// col0 + ncols)), row-major in the exchange buffer at `off`; only the pairs
// row < col are copied (the rest is padding, never unpacked).  Consecutive
// blocks of one footprint part with one destination are merged and pieces of
// more than PIECE_MAX values split, identically on both sides.
#pragma once

#include <cstdint>

#include "mp_device.cuh"

namespace mp {

struct PieceDesc {
    int32_t row0, nrows, col0, ncols;
    int64_t off;  // offset in the rank's send (pack) or receive (unpack) buffer
};

constexpr int64_t PIECE_MAX = 1 << 16;  // values per piece (one CTA each)

// PACK: x -> buf.  !PACK: buf -> x.  One CTA per piece.
template <bool PACK>
__global__ void __launch_bounds__(256) piece_copy_kernel(const PieceDesc *pd, double *x, int64_t ld,
                                                         double *buf) {
    const PieceDesc p = pd[blockIdx.x];
    double *base = buf + p.off;
    const int cnt = p.nrows * p.ncols;  // <= PIECE_MAX
    for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
        const int r = e / p.ncols, c = e - r * p.ncols;
        const int row = p.row0 + r, col = p.col0 + c;
        if (row >= col) continue;
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
