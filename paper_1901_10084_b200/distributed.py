"""Multi-GPU host logic.

One instance over several GPUs: the tiles of a round are conflict-free, so
they are spread over ranks (``shard_rounds``: longest-processing-time per
round; the library's ``mp_shard_plan`` computes the same plan).  Each tile
always runs on the same rank, which keeps its duals; after every round a
rank sends each grid block of its tiles' *footprints* (``tile_footprint``: the
pairs a tile writes back) to the rank whose tile touches that block next
(``next_toucher``), and a block's last toucher of the pass sends it to every
rank, so every tile reads the single-GPU x and every rank enters the pair
phase with it.  ``ShardedSession`` is one rank of that (one process per GPU,
grouped NCCL send/recv inside the library); ``LocalShardGroup`` drives all
ranks of one instance from one process on one device through the same
per-round code, with device copies as the transport -- the single-GPU test
harness.

``bench.py`` under torchrun runs config 4 (n = 10000) sharded over all ranks
(strong scaling); ``--replicas`` measures independent instances instead
(DESIGN.md section 6).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import schedule


@dataclass(frozen=True)
class DistEnv:
    world: int
    rank: int
    local_rank: int


def dist_env() -> DistEnv:
    return DistEnv(int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
                   int(os.environ.get("LOCAL_RANK", "0")))


def max_over_ranks(value: float, device=None) -> float:
    """All-reduce MAX of a float (a no-op without an initialised group)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def shard_rounds(n: int, b: int, world: int):
    """Per round, a list of (tile index in round, rank): longest-processing-
    time assignment by triplet count, so each round's slowest GPU is as
    light as possible (LPT ~0.96-0.998 efficiency)."""
    plan = []
    for rnd in schedule.tiled_rounds(n, b):
        loads = [0] * world
        order = sorted(range(len(rnd.units)), key=lambda t: -rnd.units[t].size)
        assign = {}
        for t in order:
            g = min(range(world), key=lambda r: (loads[r], r))
            assign[t] = g
            loads[g] += rnd.units[t].size
        plan.append([(t, assign[t]) for t in range(len(rnd.units))])
    return plan


def balance_efficiency(n: int, b: int, world: int) -> float:
    """ideal / achieved of sum over rounds of the per-round max rank load."""
    rounds = schedule.tiled_rounds(n, b)
    plan = shard_rounds(n, b, world)
    total = crit = 0
    for rnd, asg in zip(rounds, plan):
        loads = [0] * world
        for t, g in asg:
            loads[g] += rnd.units[t].size
        total += sum(loads)
        crit += max(loads) if loads else 0
    return (total / world) / crit if crit else 1.0


def exchange_volume(n: int, b: int, world: int):
    """Pairs each rank must receive before each round: pairs its round-r
    tiles touch whose last writer (an earlier round) was another rank.
    Returns the per-round totals (small n only: enumerates triplets)."""
    rounds = schedule.tiled_rounds(n, b)
    plan = shard_rounds(n, b, world)
    owner = {}
    volume = []
    for rnd, asg in zip(rounds, plan):
        need = 0
        touched = []
        for t, g in asg:
            pairs = set()
            for (i, j, k) in schedule.tile_triplets(rnd.units[t], n):
                pairs.update(((i, j), (i, k), (j, k)))
            need += sum(1 for p in pairs if p in owner and owner[p] != g)
            touched.append((pairs, g))
        for pairs, g in touched:
            for p in pairs:
                owner[p] = g
        volume.append(need)
    return volume


# ---------------------------------------------------------------------------
# footprints (what a tile writes back; mp_shard.cuh)
# ---------------------------------------------------------------------------

def tile_footprint(tile, n):
    """Pairs tile ``tile`` writes back (mp_device.cuh ring_block / rk_block):
    R x J with j < klo, R x K, and J x K with j > ihi, each with first < second."""
    ilo, ihi = tile.rows
    klo, z = tile.cols
    jlo, jhi = tile.middle
    out = set()
    for i in range(ilo, ihi + 1):
        for j in range(max(jlo, i + 1), min(jhi, klo - 1) + 1):
            out.add((i, j))
        for k in range(max(klo, i + 1), z + 1):
            out.add((i, k))
    for j in range(max(jlo, ihi + 1), jhi + 1):
        for k in range(max(klo, j + 1), z + 1):
            out.add((j, k))
    return {(i, j) for (i, j) in out if j <= n - 1}


# ---------------------------------------------------------------------------
# next-toucher routing (who needs a footprint block next; mp_shard.cuh)
# ---------------------------------------------------------------------------
# Tiles and pairs live on one global grid: row block I holds rows
# [1 + (I-1) b, I b] (I = 0: row 0 alone -- every tile has x = 1 - b + I b) and
# column block K the columns [n - b - K b, n - 1 - K b] (every tile has
# z = n - 1 - K b).  Tile (I, K) runs in round K - I of the first family when
# K >= I, else in round I - 1 - K of the second (schedule.tiled_rounds).  Its
# footprint is the union of whole grid blocks (the pairs p < q of each): its RK
# block (I, K), the WR blocks (I, K') with K' > K down to the diagonal, and the
# WK blocks (I', K) with I' > I down to the diagonal.  Conversely block (Ia, Kb)
# is touched by the tiles of row Ia with K <= Kb and the tiles of column Kb with
# I <= Ia, each of which touches all of its pairs, in the schedule order that
# ``block_touchers`` lists.  A tile's blocks therefore go to one or two
# neighbour tiles (the next tile of its row, the next of its column); a
# block's last toucher of the pass sends it to every rank (the pair phase
# runs on all of them).

def tile_block(n, b, tile):
    return (tile.x + b - 1) // b, (n - 1 - tile.z) // b


def block_tile(n, b, I, K):
    """The tile of row block I and column block K, or None."""
    x, z = 1 - b + I * b, n - 1 - K * b
    if I < 0 or K < 0 or z < max(x, 0) + 2:
        return None
    return schedule.Tile(x, z, b)


def tile_round(n, b, I, K):
    """(round index, position in the round) of tile (I, K)."""
    r1 = len(range(n - 1, 1, -b))
    return (K - I, I) if K >= I else (r1 + I - 1 - K, K)


def row_block(b, r):
    return 0 if r <= 0 else (r + b - 1) // b


def col_block(n, b, c):
    return (n - 1 - c) // b


def block_touchers(n, b, Ia, Kb):
    """Tiles touching grid block (Ia, Kb), in schedule order."""
    if Kb >= Ia:
        seq = ([(Ia, k) for k in range(Ia, Kb + 1)] + [(i, Kb) for i in range(Ia - 1, -1, -1)]
               + [(Ia, k) for k in range(Ia - 1, -1, -1)])
    else:
        seq = ([(i, Kb) for i in range(Kb, -1, -1)] + [(i, Kb) for i in range(Kb + 1, Ia + 1)]
               + [(Ia, k) for k in range(Kb - 1, -1, -1)])
    return [t for t in seq if block_tile(n, b, *t) is not None]


def next_toucher(n, b, Ia, Kb, I, K):
    """The tile touching block (Ia, Kb) next after tile (I, K) in this pass
    (closed form of ``block_touchers``), or None when (I, K) is the last."""
    def first(cands):
        for t in cands:
            if block_tile(n, b, *t) is not None:
                return t
        return None
    tail = Ia if Kb >= Ia else Kb       # the closing run (Ia, tail-1 .. 0) of the row
    if I == Ia and K < tail:            # inside the closing run
        return (Ia, K - 1) if K >= 1 else None
    if Kb >= Ia:
        if I == Ia:                     # opening run of the row: K in [Ia, Kb]
            if K < Kb:                  # (only the block's own tile may be missing)
                return first([(Ia, K + 1), (Ia - 1, Kb)] if Ia >= 1 else [(Ia, K + 1)])
            return (Ia - 1, Kb) if Ia >= 1 else None
        # column run, I falling from Ia - 1 to 0, then the closing run
        return (I - 1, Kb) if I >= 1 else ((Ia, Ia - 1) if Ia >= 1 else None)
    if I <= Kb and K == Kb:             # column run of the first family, I falling
        return (I - 1, Kb) if I >= 1 else first([(Kb + 1, Kb)] + ([(Ia, Kb - 1)] if Kb >= 1 else []))
    if K == Kb and I < Ia:              # column run of the second family, I rising
        return first([(I + 1, Kb)] + ([(Ia, Kb - 1)] if Kb >= 1 else []))
    return (Ia, Kb - 1) if Kb >= 1 else None   # the block's own tile


def footprint_blocks(n, b, I, K):
    """Grid blocks of tile (I, K)'s footprint: [("RK" | "WR" | "WK", Ia, Kb)]."""
    t = block_tile(n, b, I, K)
    ilo, ihi = t.rows
    klo, z = t.cols
    jlo, jhi = t.middle
    out = [("RK", I, K)]
    wr0, wr1 = max(jlo, ilo + 1), min(jhi, klo - 1)
    if wr1 >= wr0:
        out += [("WR", I, kb) for kb in range(col_block(n, b, wr1), col_block(n, b, wr0) + 1)]
    wk0 = max(jlo, ihi + 1)
    if jhi >= wk0:
        out += [("WK", ia, K) for ia in range(row_block(b, wk0), row_block(b, jhi) + 1)]
    return out


def block_pairs(n, b, Ia, Kb):
    r0, r1 = (0, 0) if Ia == 0 else (1 + (Ia - 1) * b, Ia * b)
    c0, c1 = max(n - b - Kb * b, 0), n - 1 - Kb * b
    return {(p, q) for p in range(r0, min(r1, n - 1) + 1) for q in range(max(c0, p + 1), c1 + 1)}


def route_volumes(n, b, world, owner=None, broadcast=True):
    """Pairs sent per round under next-toucher routing: a list (one entry per
    round) of world x world matrices vol[src][dst]; a block whose next toucher
    runs on another rank goes to that rank only, a block's last toucher of the
    pass sends it to every other rank (``broadcast=False`` leaves those out:
    what remains is exactly ``exchange_volume``'s need).  ``owner[(I, K)]``
    defaults to the LPT plan."""
    rounds = schedule.tiled_rounds(n, b)
    if owner is None:
        owner = {}
        for rnd, asg in zip(rounds, shard_rounds(n, b, world)):
            for t, g in asg:
                owner[tile_block(n, b, rnd.units[t])] = g
    out = []
    for rnd in rounds:
        vol = np.zeros((world, world), dtype=np.int64)
        for tile in rnd.units:
            I, K = tile_block(n, b, tile)
            src = owner[(I, K)]
            for _, ia, kb in footprint_blocks(n, b, I, K):
                cnt = len(block_pairs(n, b, ia, kb))
                nxt = next_toucher(n, b, ia, kb, I, K)
                if nxt is None:
                    for d in range(world if broadcast else 0):
                        if d != src:
                            vol[src, d] += cnt
                elif owner[nxt] != src:
                    vol[src, owner[nxt]] += cnt
        out.append(vol)
    return out


def merge_duals(parts):
    """Merge per-shard (keys, vals, order) into the single-worker visit order:
    entries of one tile live on one shard and are already in order, so a
    stable sort on the tile's schedule index is enough."""
    keys = np.concatenate([p[0] for p in parts]) if parts else np.empty(0, np.int64)
    vals = np.concatenate([p[1] for p in parts]) if parts else np.empty(0)
    order = np.concatenate([p[2] for p in parts]) if parts else np.empty(0, np.int64)
    idx = np.argsort(order, kind="stable")
    return keys[idx], vals[idx]


def native_shard_plan(n, b, world):
    """Tile owners of the library's LPT plan in schedule order (host only)."""
    from . import _native
    L = _native.load()
    cnt = ctypes.c_int64()
    _native.check(L.mp_shard_plan(n, b, world, None, ctypes.byref(cnt)), "mp_shard_plan")
    owner = np.empty(cnt.value, dtype=np.int32)
    _native.check(L.mp_shard_plan(n, b, world, owner.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                  ctypes.byref(cnt)), "mp_shard_plan")
    return owner


def native_route_volumes(n, b, world):
    """The library's exchange plan (host only): per round a world x world
    matrix of pairs sent, ``route_volumes``'s twin."""
    from . import _native
    L = _native.load()
    nr = ctypes.c_int64()
    _native.check(L.mp_shard_route(n, b, world, None, ctypes.byref(nr)), "mp_shard_route")
    vol = np.zeros((nr.value, world, world), dtype=np.int64)
    _native.check(L.mp_shard_route(n, b, world, _native.iptr(vol), ctypes.byref(nr)), "mp_shard_route")
    return vol


# ---------------------------------------------------------------------------
# sharded execution
# ---------------------------------------------------------------------------

class LocalShardGroup:
    """All ``world`` ranks of one sharded solve as sessions of this process on
    one device, run together by ``mp_group_run_passes`` (exchange by device
    copies).  Bitwise equal to a single session by construction; used to test
    the sharded path without several GPUs."""

    def __init__(self, instance, world, tile_size=40, schedule_kind="tiled", device=0):
        from .solver import DeviceSession
        self.world = world
        self.members = [DeviceSession(instance, schedule_kind, tile_size, device)
                        for _ in range(world)]
        for g, s in enumerate(self.members):
            s.shard(world, g)

    def run(self, npasses=1):
        from . import _native
        from .solver import SolverError
        out = (_native.MPPassStats * max(npasses, 1))()
        hs = (ctypes.c_void_p * self.world)(*[s._h for s in self.members])
        rc = _native.load().mp_group_run_passes(hs, self.world, npasses, out)
        if rc == _native.MP_ERR_NONFINITE:
            raise SolverError(_native.last_error())
        _native.check(rc, "mp_group_run_passes")
        return list(out)[:npasses]

    def state(self, member=0):
        return self.members[member].state()

    def duals(self):
        return merge_duals([s.duals_ranked() for s in self.members])

    def set_duals(self, keys, vals, pair_duals=None):
        for s in self.members:
            s.set_duals(keys, vals, pair_duals)

    def close(self):
        for s in self.members:
            s.close()


class ShardedSession:
    """This process's rank of a sharded solve (one process per GPU; the NCCL
    communicator is created inside the library from an id that rank 0 makes
    and ``torch.distributed`` broadcasts)."""

    def __init__(self, instance, tile_size=40, schedule_kind="tiled", device=None):
        import torch.distributed as dist
        from . import _native
        from .solver import DeviceSession
        env = dist_env()
        self.world, self.rank = env.world, env.rank
        dev = env.local_rank if device is None else device
        self.session = DeviceSession(instance, schedule_kind, tile_size, dev)
        uid = [None]
        if self.rank == 0:
            buf = ctypes.create_string_buffer(128)
            _native.check(_native.load().mp_nccl_unique_id(buf), "mp_nccl_unique_id")
            uid[0] = buf.raw
        if self.world > 1:
            dist.broadcast_object_list(uid, src=0)
        self.session.shard(self.world, self.rank, uid[0])

    def run(self, npasses=1):
        return self.session.run(npasses)

    def state(self):
        return self.session.state()

    def duals(self):
        """Global duals in visit order (collective: every rank must call)."""
        import torch.distributed as dist
        part = self.session.duals_ranked()
        parts = [None] * self.world
        if self.world > 1:
            dist.all_gather_object(parts, part)
        else:
            parts = [part]
        return merge_duals(parts)

    def close(self):
        self.session.close()
