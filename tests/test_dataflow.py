"""The dataflow launch's dependency rules (mp_device.cuh, DF_*), checked
exhaustively on CPU against the per-pair last toucher of the whole tiled
schedule (schedule.tiled_rounds, schedule.py:117-153):

for every tile (x, z) of the second family (the rounds (x + c*b, n-1 - c*b),
x >= 1) and every pair it
touches, the tile that touched the pair last in the reference order is a
first-family tile (finished before the launch), none, the row predecessor
(x, z - b) or the column predecessor (x - b, z); pairs from the row
predecessor are this tile's x_ij (rows R, columns below klo) and lie in the
predecessor's WR ring (columns below its klo) or, for columns in
[klo - b, klo), in its RK block; pairs from the column predecessor are in
this tile's columns K with rows above the predecessor's rows (its WK ring).
One exception, near the diagonal: a tile with z - x = b + 1 (rows and
columns overlapping) may read pairs its row predecessor never touched, last
touched by the diagonal predecessor (x - b, z - b) two rounds back; the
device waits for that tile to finish before such a tile starts (DF_DIAG).
"""

import pytest

from paper_1901_10084_b200 import schedule


def touched(t, b):
    """Pairs (a, c), a < c, tile t touches, in any role (_kernels.py:74-131)."""
    ilo, ihi = max(t.x, 0), t.x + b - 1
    klo, z = max(t.z - b + 1, 0), t.z
    jlo, jhi = max(t.x + 1, 1), z - 1
    out = set()
    for i in range(ilo, ihi + 1):
        for j in range(max(jlo, i + 1), jhi + 1):
            for k in range(max(klo, j + 1), z + 1):
                out.update(((i, j), (i, k), (j, k)))
    return out


@pytest.mark.parametrize("n,b", [(9, 2), (14, 3), (23, 4), (31, 5), (40, 8), (57, 6), (19, 1), (64, 7),
                                 (130, 40), (173, 40)])
def test_second_family_predecessors(n, b):
    rounds = [r for r in schedule.tiled_rounds(n, b) if r.units]
    # the second family: the rounds from the first one whose first tile has x >= 1
    r0 = next(i for i, r in enumerate(rounds) if r.units[0].x >= 1)
    fam2 = {(t.x, t.z) for r in rounds[r0:] for t in r.units}
    last = {}  # pair -> (x, z) of the last tile that touched it
    checked = diag_seen = 0
    for ri, rnd in enumerate(rounds):
        cur = []
        for t in rnd.units:
            pairs = touched(t, b)
            if ri >= r0:
                row_pred, col_pred = (t.x, t.z - b), (t.x - b, t.z)
                diag_pred = (t.x - b, t.z - b) if t.z - t.x <= 2 * b else None
                ilo, klo = t.x, max(t.z - b + 1, 0)
                for (a, c) in pairs:
                    p = last.get((a, c))
                    if p is None or p not in fam2:  # untouched, or first family
                        continue
                    assert p in (row_pred, col_pred, diag_pred), ((n, b), (t.x, t.z), (a, c), p)
                    if p == diag_pred:
                        diag_seen += 1
                    elif p == row_pred:
                        assert ilo <= a <= t.x + b - 1 and c < klo
                        pk = max(p[1] - b + 1, 0)
                        if c >= klo - b:   # the predecessor's RK block: written at its end
                            assert pk <= c <= p[1]
                        else:              # its WR ring
                            assert c < pk
                    else:
                        assert klo <= c <= t.z and a > p[0] + b - 1  # its WK ring (rows > its ihi)
                    checked += 1
            cur.append(((t.x, t.z), pairs))
        for key, pairs in cur:  # tiles of a round touch disjoint pairs
            for pr in pairs:
                last[pr] = key
    assert checked > 0 or n < 4 * b


def test_second_family_predecessors_sweep():
    """Every small shape: b = 1..9, n up to 62."""
    for b in range(1, 10):
        for n in range(5, 63, 7):
            test_second_family_predecessors(n, b)
