"""Conflict-free schedule of the triplet set and its mapping onto CTAs.

Host mirror of the reference's ``schedule.py`` (same public names) plus the
B200 mapping the native library uses:

* a **round** (``Round``) is one anti-diagonal of b x b tiles of S_{i,k}
  sets; tiles of one round share no pair (schedule.py:235-250) -> one kernel
  launch per round, one CTA per tile;
* inside a tile the CTA sweeps the **levels** L = i+j+k (``tile_levels``);
  same-level triplets never share a pair, and the reference visits
  conflicting triplets in increasing L, so the sweep reproduces the
  reference order exactly.

The native library builds the same schedule in C++ (``mp_solver.cu``,
``mp_create``); tests compare the two.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass


@dataclass(frozen=True)
class TripletSet:
    """S_{i,k} = {(i, j, k) : i < j < k} (schedule.py:17-33)."""
    i: int
    k: int

    def __post_init__(self):
        if self.k < self.i + 2:
            raise ValueError(f"S_({self.i},{self.k}) is empty; need k >= i + 2")

    @property
    def size(self):
        return self.k - self.i - 1

    def triplets(self):
        return ((self.i, j, self.k) for j in range(self.i + 1, self.k))


@dataclass(frozen=True)
class Tile:
    """b x b block of S_{i,k}: i in [x, x+b-1], k in [z-b+1, z], clipped to
    the valid range (schedule.py:36-67)."""
    x: int
    z: int
    b: int

    def __post_init__(self):
        if self.b < 1:
            raise ValueError(f"tile size must be >= 1, got {self.b}")
        if self.z < max(self.x, 0) + 2:
            raise ValueError(f"tile ({self.x},{self.z}) contains no triplets")

    @property
    def rows(self):
        return max(self.x, 0), self.x + self.b - 1

    @property
    def cols(self):
        return max(self.z - self.b + 1, 0), self.z

    @property
    def middle(self):
        return max(self.x + 1, 1), self.z - 1

    def sets(self):
        ilo, ihi = self.rows
        klo, khi = self.cols
        return [TripletSet(i, k) for i in range(ilo, ihi + 1)
                for k in range(max(klo, i + 2), khi + 1)]

    @property
    def size(self):
        return sum(s.size for s in self.sets())

    def levels(self):
        """Inclusive range of L = i+j+k over the tile's triplets."""
        ilo, ihi = self.rows
        klo, z = self.cols
        jlo, _ = self.middle
        j0 = max(jlo, ilo + 1)
        k0 = max(klo, j0 + 1)
        return ilo + j0 + k0, min(ihi, z - 2) + (z - 1) + z


@dataclass(frozen=True)
class Round:
    """Mutually independent units; unit at 0-based position r goes to worker
    (r+1) mod p (schedule.py:70-84)."""
    units: tuple

    def worker_of(self, position, p):
        return (position + 1) % p

    @property
    def size(self):
        return sum(u.size for u in self.units)


def _anti_diagonal(x, z, b):
    out = []
    c = 0
    while max(x + c * b, 0) + 2 <= z - c * b:
        out.append(Tile(x + c * b, z - c * b, b))
        c += 1
    return out


def tiled_rounds(n, b):
    """Block anti-diagonals of the (i, k) grid (schedule.py:117-153): first
    z = n-1, n-1-b, ... with x = 1-b, then x = 1, 1+b, ... with z = n-1."""
    if n < 3:
        raise ValueError(f"need n >= 3, got {n}")
    if b < 1:
        raise ValueError(f"tile size must be >= 1, got {b}")
    starts = [(1 - b, z) for z in range(n - 1, 1, -b)]
    starts += [(x, n - 1) for x in range(1, n - 2, b)]
    return [Round(tuple(_anti_diagonal(x, z, b))) for x, z in starts]


def diagonal_rounds(n):
    """Anti-diagonals of single S_{i,k} sets (schedule.py:94-114)."""
    if n < 3:
        raise ValueError(f"need n >= 3, got {n}")
    out = []
    for x, z in [(0, z) for z in range(n - 1, 1, -1)] + [(x, n - 1) for x in range(1, n - 2)]:
        out.append(Round(tuple(TripletSet(x + c, z - c) for c in range((z - x - 2) // 2 + 1))))
    return out


def tile_triplets(tile, n):
    """Reference cube order inside a tile (schedule.py:156-175)."""
    x, z, b = tile.x, tile.z, tile.b
    if z > n - 1:
        raise ValueError(f"tile ({x},{z}) out of range for n={n}")
    klo, _ = tile.cols
    ilo, ihi = tile.rows
    for jb in range(x + 1, z, b):
        je = min(jb + b - 1, z - 1)
        for k in range(klo, z + 1):
            for j in range(max(jb, 1), min(je, k - 1) + 1):
                for i in range(ilo, min(ihi, j - 1) + 1):
                    yield (i, j, k)


def unit_triplets(unit, n):
    return tile_triplets(unit, n) if isinstance(unit, Tile) else unit.triplets()


def tile_level_order(tile, n):
    """The device's order inside a tile: by level L, then by slot of the
    (i, k) pair.  A linear extension of ``tile_triplets``'s conflict order."""
    trips = list(tile_triplets(tile, n))
    ilo, _ = tile.rows
    klo, _ = tile.cols
    return sorted(trips, key=lambda t: (sum(t), (t[0] - ilo) * tile.b + (t[2] - klo)))


def verify_partition(rounds, n):
    """Every triplet in exactly one unit (schedule.py:222-232)."""
    seen = [t for rnd in rounds for u in rnd.units for t in unit_triplets(u, n)]
    expected = n * (n - 1) * (n - 2) // 6
    return len(seen) == expected and len(set(seen)) == expected


def verify_independence(rounds, n):
    """Units of one round touch disjoint pairs (schedule.py:235-250)."""
    for rnd in rounds:
        owner = {}
        for u_idx, unit in enumerate(rnd.units):
            for (i, j, k) in unit_triplets(unit, n):
                for pr in ((i, j), (i, k), (j, k)):
                    if owner.setdefault(pr, u_idx) != u_idx:
                        return False
    return True


# ---------------------------------------------------------------------------
# schedule depth
# ---------------------------------------------------------------------------

def critical_levels(n, b):
    """Barrier depth of a pass: sum over rounds of the deepest tile's level
    count (the device runs the second family as one dataflow
    launch, whose depth is far smaller, see tests/test_dataflow.py)."""
    total = 0
    for rnd in tiled_rounds(n, b):
        if rnd.units:
            total += max(hi - lo + 1 for lo, hi in (t.levels() for t in rnd.units))
    return total


# ---------------------------------------------------------------------------
# algorithmic traffic
# ---------------------------------------------------------------------------

def _tile_arrays(n, b):
    xs, zs = [], []
    for x0, z0 in [(1 - b, z) for z in range(n - 1, 1, -b)] + [(x, n - 1) for x in range(1, n - 2, b)]:
        c = 0
        while max(x0 + c * b, 0) + 2 <= z0 - c * b:
            xs.append(x0 + c * b)
            zs.append(z0 - c * b)
            c += 1
    import numpy as np
    return np.array(xs, dtype=np.int64), np.array(zs, dtype=np.int64)


def touched_pairs(n, b, chunk=2048):
    """T_x(n, b): sum over all tiles of a pass of the distinct pairs the tile
    touches (R x J, J x K, R x K with i < j < k), i.e. the pairs one pass
    must read and write once each under the tiled schedule."""
    import numpy as np
    X, Z = _tile_arrays(n, b)
    total = 0
    ar = np.arange(b, dtype=np.int64)
    for s in range(0, len(X), chunk):
        x, z = X[s:s + chunk, None], Z[s:s + chunk, None]
        ilo, ihi = np.maximum(x, 0), x + b - 1
        klo = np.maximum(z - b + 1, 0)
        jlo, jhi = np.maximum(x + 1, 1), z - 1
        i = ilo + ar[None, :]                       # (T, b) rows
        k = klo + ar[None, :]                       # (T, b) cols
        iv = (i <= ihi) & (i <= n - 1)
        kv = k <= z
        # R x J with j outside K (j < klo)
        wr = np.clip(np.minimum(jhi, klo - 1) - np.maximum(jlo, i + 1) + 1, 0, None)
        total += int((wr * iv).sum())
        # J x K with j outside R (j > ihi)
        wk = np.clip(np.minimum(jhi, k - 1) - np.maximum(jlo, ihi + 1) + 1, 0, None)
        total += int((wk * kv).sum())
        # R x K pairs touched in any role
        I, K = i[:, :, None], k[:, None, :]
        JLO, JHI, ILO = jlo[:, :, None], jhi[:, :, None], ilo[:, :, None]
        valid = iv[:, :, None] & kv[:, None, :] & (I < K)
        as_ik = np.maximum(I + 1, JLO) <= np.minimum(K - 1, JHI)
        as_ij = (K >= JLO) & (K <= JHI)
        as_jk = (I >= JLO) & (I <= JHI) & (I > ILO)
        total += int((valid & (as_ik | as_ij | as_jk)).sum())
    return total


def touched_pairs_brute(n, b):
    """Reference count by enumeration (small n only)."""
    total = 0
    for rnd in tiled_rounds(n, b):
        for t in rnd.units:
            s = set()
            for (i, j, k) in tile_triplets(t, n):
                s.update(((i, j), (i, k), (j, k)))
            total += len(s)
    return total
