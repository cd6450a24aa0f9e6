"""Multi-GPU host logic.

Today ``bench.py --gpus N`` runs N independent replicas (one solve per GPU,
weak scaling) and reports the whole-box rate from the max-over-ranks device
time.  The sharded single-instance path of SURVEY.md 8(e) -- tiles of one
round spread over GPUs, duals local, touched x exchanged between rounds --
is planned here (``shard_rounds`` / ``exchange_volume``) and validated on
CPU; its device execution is future work.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

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
