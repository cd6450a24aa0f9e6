"""Multi-GPU host logic.

One instance over several GPUs: the tiles of a round are conflict-free, so
they are spread over ranks (``shard_rounds``: longest-processing-time per
round; the library's ``mp_shard_plan`` computes the same plan).  Each tile
always runs on the same rank, which keeps its duals; after every round the
ranks exchange the *footprints* of their tiles (``tile_footprint``: the pairs
a tile writes back) so every rank holds the single-GPU x before the next
round.  ``ShardedSession`` is one rank of that (one process per GPU, NCCL
all-gather inside the library); ``LocalShardGroup`` drives all ranks of one
instance from one process on one device through the same per-round code, with
device copies as the transport -- the single-GPU test harness.

``bench.py --gpus N`` measures N independent replicas (weak scaling, one
config-2 instance per GPU): at n = 1000 a round has at most 13 tiles, so one
instance cannot use more than one GPU.
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
