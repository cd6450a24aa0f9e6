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


def serial_order(n):
    if n < 3:
        raise ValueError(f"need n >= 3, got {n}")
    return itertools.combinations(range(n), 3)


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


class WorkerPlan:
    """Static assignment of round units to workers (schedule.py:184-215)."""

    def __init__(self, rounds, p):
        if p < 1:
            raise ValueError(f"need at least one worker, got {p}")
        self.p = p
        self.rounds = rounds
        self.by_round = []
        for rnd in rounds:
            lanes = [[] for _ in range(p)]
            for pos, unit in enumerate(rnd.units):
                lanes[rnd.worker_of(pos, p)].append(unit)
            self.by_round.append(lanes)

    def worker_units(self, w):
        for lanes in self.by_round:
            yield from lanes[w]

    def worker_triplets(self, w, n):
        for unit in self.worker_units(w):
            yield from unit_triplets(unit, n)

    def worker_load(self, w):
        return sum(u.size for u in self.worker_units(w))


def worker_plan(rounds, p):
    return WorkerPlan(rounds, p)


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
# device mapping (mirrors mp_create in csrc/mp_solver.cu)
# ---------------------------------------------------------------------------

def _max_threads(slots):
    return 1024 if slots == 1 else (832 if slots == 2 else 768)


def cta_shape(b):
    """(slots per thread S, threads per CTA) for tile size b."""
    s = 1
    while True:
        nt = ((b * b + s - 1) // s + 31) // 32 * 32
        if nt <= _max_threads(s):
            return s, nt
        s += 1


def launch_plan(n, b):
    """Per round, the CTAs of its launch: list of lists of (x, z, Lbeg, Lend)."""
    return [[(t.x, t.z, *t.levels()) for t in rnd.units] for rnd in tiled_rounds(n, b)]


def critical_levels(n, b):
    """Sum over rounds of the deepest tile's level count: the number of
    dependent __syncthreads() steps in one pass."""
    total = 0
    for rnd in tiled_rounds(n, b):
        if rnd.units:
            total += max(hi - lo + 1 for lo, hi in (t.levels() for t in rnd.units))
    return total
