"""Multi-rank host logic on CPU with gloo (world_size 2)."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_1901_10084_b200 import distributed, schedule


def test_shard_plan_covers_every_tile_once():
    for n, b, g in [(60, 8, 2), (100, 40, 4), (200, 16, 8)]:
        plan = distributed.shard_rounds(n, b, g)
        rounds = schedule.tiled_rounds(n, b)
        for rnd, asg in zip(rounds, plan):
            assert sorted(t for t, _ in asg) == list(range(len(rnd.units)))
            assert all(0 <= r < g for _, r in asg)
        assert 0 < distributed.balance_efficiency(n, b, g) <= 1.0


def test_lpt_balance_improves_with_n():
    assert distributed.balance_efficiency(2000, 40, 8) > distributed.balance_efficiency(400, 40, 8)
    assert distributed.balance_efficiency(2000, 40, 2) > 0.9


def test_exchange_volume_single_rank_is_zero():
    assert sum(distributed.exchange_volume(40, 5, 1)) == 0
    assert sum(distributed.exchange_volume(40, 5, 2)) > 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    env = distributed.dist_env()
    t = distributed.max_over_ranks(1.5 + rank)  # bench.py: max-over-ranks device time
    plan = distributed.shard_rounds(64, 8, world)  # every rank derives the same plan
    import torch
    import hashlib
    h = torch.tensor([int(hashlib.sha256(str(plan).encode()).hexdigest()[:12], 16)],
                     dtype=torch.int64)
    hs = [torch.zeros_like(h) for _ in range(world)]
    dist.all_gather(hs, h)
    q.put((env.rank, env.world, t, len({int(x) for x in hs})))
    dist.destroy_process_group()


def test_gloo_two_ranks_max_timing_and_consistent_plan():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert [o[0] for o in out] == [0, 1]
    assert all(o[1] == 2 and o[2] == 2.5 and o[3] == 1 for o in out)
