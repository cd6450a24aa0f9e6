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


# ---------------------------------------------------------------------------
# sharded execution: plan, footprints, dual merge (host logic of mp_shard)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("n,b,world", [(60, 8, 2), (100, 40, 4), (200, 16, 8), (333, 12, 3)])
def test_native_plan_matches_python_plan(n, b, world):
    owner = distributed.native_shard_plan(n, b, world)
    py = [g for asg in distributed.shard_rounds(n, b, world) for _, g in asg]
    assert owner.tolist() == py


@pytest.mark.parametrize("n,b", [(17, 3), (30, 8), (41, 5), (25, 40)])
def test_footprints_cover_touched_pairs_and_are_disjoint(n, b):
    for rnd in schedule.tiled_rounds(n, b):
        seen = set()
        for t in rnd.units:
            fp = distributed.tile_footprint(t, n)
            touched = set()
            for (i, j, k) in schedule.tile_triplets(t, n):
                touched.update(((i, j), (i, k), (j, k)))
            assert touched <= fp
            assert not (fp & seen)  # one round's footprints never overlap
            seen |= fp


@pytest.mark.parametrize("n,b", [(17, 3), (30, 8), (41, 5), (25, 40), (33, 4), (23, 1), (90, 40)])
def test_next_toucher_follows_every_pair_through_the_pass(n, b):
    """A tile's footprint is a union of whole grid blocks, every toucher of a
    block touches all of its pairs, and the closed-form next toucher is the
    next tile that touches each pair in schedule order (the last one has
    none): what the sharded exchange routes by (mp_shard.cuh)."""
    D = distributed
    last = {}
    for rnd in schedule.tiled_rounds(n, b):
        for t in rnd.units:
            I, K = D.tile_block(n, b, t)
            assert D.block_tile(n, b, I, K) == t
            fp = D.tile_footprint(t, n)
            union = set()
            for _, ia, kb in D.footprint_blocks(n, b, I, K):
                pairs = D.block_pairs(n, b, ia, kb)
                assert pairs and not (union & pairs)
                union |= pairs
                seq = D.block_touchers(n, b, ia, kb)
                pos = seq.index((I, K))
                assert D.next_toucher(n, b, ia, kb, I, K) == (seq[pos + 1] if pos + 1 < len(seq) else None)
            assert union == fp
            for p in fp:
                blk = (D.row_block(b, p[0]), D.col_block(n, b, p[1]))
                if p in last:
                    assert D.next_toucher(n, b, *blk, *last[p]) == (I, K)
                else:
                    assert D.block_touchers(n, b, *blk)[0] == (I, K)
                last[p] = (I, K)
    assert len(last) == n * (n - 1) // 2
    for p, t in last.items():
        assert D.next_toucher(n, b, D.row_block(b, p[0]), D.col_block(n, b, p[1]), *t) is None


@pytest.mark.parametrize("n,b,world", [(60, 8, 2), (100, 40, 4), (200, 16, 8), (45, 6, 3), (23, 1, 2)])
def test_native_route_matches_python_route(n, b, world):
    import numpy as np
    py = np.array(distributed.route_volumes(n, b, world))
    nat = distributed.native_route_volumes(n, b, world)
    assert py.shape == nat.shape and np.array_equal(py, nat)
    assert all(nat[r][g][g] == 0 for r in range(len(nat)) for g in range(world))


@pytest.mark.parametrize("n,b,world", [(40, 5, 2), (60, 8, 3), (64, 8, 4)])
def test_route_volume_is_the_need_plus_one_broadcast(n, b, world):
    """Without the end-of-pass broadcasts the routed volume is exactly what
    the ranks need (exchange_volume: pairs whose last writer was another
    rank); the broadcasts add each pair once per other rank; an all-gather of
    every footprint would move (world - 1) copies of every touched pair."""
    import numpy as np
    need = sum(distributed.exchange_volume(n, b, world))
    routed = int(np.array(distributed.route_volumes(n, b, world, broadcast=False)).sum())
    assert routed == need
    total = int(np.array(distributed.route_volumes(n, b, world)).sum())
    assert total == need + (world - 1) * (n * (n - 1) // 2)
    gathered = (world - 1) * schedule.touched_pairs_brute(n, b)
    assert total < gathered


def test_merge_duals_restores_visit_order():
    import numpy as np
    keys = np.arange(10, dtype=np.int64) * 7
    order = np.array([0, 0, 1, 1, 1, 4, 4, 5, 9, 9], dtype=np.int64)
    vals = keys * 0.5
    a = [(keys[m], vals[m], order[m]) for m in (order % 2 == 0, order % 2 == 1)]
    k, v = distributed.merge_duals(a)
    assert k.tolist() == keys.tolist() and v.tolist() == vals.tolist()


def _sharded_py_pass(n, b, world, rank, inst, x, f, duals, pair_duals, exchange, p2p):
    """One pass of rank `rank` of a sharded solve in the reference's arithmetic
    (oracle.py_pass restated per tile): own tiles only, after every round the
    blocks of its footprints to the ranks of their next touchers (stale
    elsewhere until the end-of-pass broadcast), pair rows locally (x identical
    on every rank by then)."""
    from oracle import oracle as orc
    eps = inst.epsilon
    plan = distributed.shard_rounds(n, b, world)
    rounds = schedule.tiled_rounds(n, b)
    owner = {distributed.tile_block(n, b, rnd.units[t]): g for rnd, asg in zip(rounds, plan) for t, g in asg}
    new, order, tix = {}, {}, 0
    viol = 0.0
    for rnd, asg in zip(rounds, plan):
        mine = []
        for t, g in asg:
            if g != rank:
                continue
            tile = rnd.units[t]
            mine.append(tile)
            for (i, j, k) in orc.tile_order(n, b, tile.x, tile.z):
                ps = (orc._pos(n, i, j), orc._pos(n, i, k), orc._pos(n, j, k))
                code = ((i * n + j) * n + k) * 3
                for kd, (pl, m1, m2) in enumerate(((ps[0], ps[1], ps[2]), (ps[1], ps[0], ps[2]),
                                                   (ps[2], ps[0], ps[1]))):
                    y = duals.get(code + kd, 0.0)
                    d0 = x[pl] - x[m1] - x[m2]
                    viol = max(viol, d0)
                    delta = d0 + y * 3.0 / eps
                    theta = eps * delta / 3.0 if delta > 0.0 else 0.0
                    coef = (y - theta) / eps
                    if coef != 0.0:
                        x[pl] += coef
                        x[m1] -= coef
                        x[m2] -= coef
                    if theta > 1e-15:
                        new[code + kd] = theta
                        order[code + kd] = tix + t
        # every block of the round's footprints to the rank of its next toucher
        # (all ranks when this was the block's last toucher of the pass): both
        # ends enumerate the round's tiles alike, so a receiver knows how many
        # values each sender has for it and where they go (mp_shard's plan)
        route = [[[] for _ in range(world)] for _ in range(world)]  # [src][dst] -> positions
        for t, g in asg:
            I, K = distributed.tile_block(n, b, rnd.units[t])
            for _, ia, kb in distributed.footprint_blocks(n, b, I, K):
                nxt = distributed.next_toucher(n, b, ia, kb, I, K)
                for d in (range(world) if nxt is None else [owner[nxt]]):
                    if d != g:
                        route[g][d] += [orc._pos(n, *p) for p in sorted(distributed.block_pairs(n, b, ia, kb))]
        got = p2p([x[route[rank][d]] for d in range(world)],
                  [len(route[s][rank]) for s in range(world)])
        for s_ in range(world):
            if s_ != rank and route[s_][rank]:
                x[route[s_][rank]] = got[s_]
        tix += len(rnd.units)
    viol = max(exchange(viol))
    return viol, new, order


def _shard_worker(rank, world, port, q):
    import numpy as np
    import torch.distributed as dist
    from paper_1901_10084_b200 import instances
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def exchange(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    def p2p(send, recv_counts):
        """Grouped point-to-point exchange (the library's ncclSend / ncclRecv
        group): send[d] to every other rank d, recv_counts[s] values from s."""
        import torch
        ops, bufs = [], [None] * world
        for d in range(world):
            if d == rank:
                continue
            if len(send[d]):
                ops.append(dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(send[d])), d))
            if recv_counts[d]:
                bufs[d] = torch.empty(recv_counts[d], dtype=torch.float64)
                ops.append(dist.P2POp(dist.irecv, bufs[d], d))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        return [None if t is None else t.numpy() for t in bufs]

    n, b = 14, 3
    inst = instances.random_instance(n, seed=11)
    x = np.zeros(inst.npairs)
    f = -inst.w_flat / inst.epsilon
    duals, pd = {}, np.zeros((inst.npairs, 2))
    for _ in range(3):
        viol, duals, order = _sharded_py_pass(n, b, world, rank, inst, x, f, duals, pd, exchange, p2p)
        # pair rows on every rank (identical x), as in oracle.py_pass
        for p in range(inst.npairs):
            for row in (0, 1):
                y = pd[p, row]
                d = inst.d_flat[p]
                d0 = (x[p] - f[p] - d) if row == 0 else (d - x[p] - f[p])
                delta = d0 + y * 2.0 / inst.epsilon
                theta = inst.epsilon * delta / 2.0 if delta > 0.0 else 0.0
                coef = (y - theta) / inst.epsilon
                if coef != 0.0:
                    x[p] = x[p] + coef if row == 0 else x[p] - coef
                    f[p] -= coef
                pd[p, row] = theta if theta > 1e-15 else 0.0
    parts = exchange((np.array(list(duals.keys()), dtype=np.int64),
                      np.array(list(duals.values())),
                      np.array([order[k] for k in duals], dtype=np.int64)))
    keys, vals = distributed.merge_duals(parts)
    q.put((rank, x.tobytes(), f.tobytes(), keys.tobytes(), vals.tobytes()))
    dist.destroy_process_group()


def test_gloo_sharded_protocol_equals_single_worker_oracle():
    """Two gloo ranks run the sharded protocol (plan, own tiles, after every
    round a grouped point-to-point exchange of the footprint blocks routed to
    their next touchers -- counts and positions derived on both ends from the
    plan, as mp_shard does -- dual merge); x, f and the merged duals equal the
    reference-order oracle bit for bit on both ranks."""
    import numpy as np
    from oracle import oracle as orc
    from paper_1901_10084_b200 import instances
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    n, b = 14, 3
    inst = instances.random_instance(n, seed=11)
    x = np.zeros(inst.npairs)
    f = -inst.w_flat / inst.epsilon
    ones = np.ones(inst.npairs)
    duals, pd = {}, np.zeros((inst.npairs, 2))
    for _ in range(3):
        _, duals = orc.py_pass(n, inst.epsilon, x, f, inst.d_flat, ones, ones, duals, pd,
                               kind="tiled", b=b)
    for r in res:
        assert np.frombuffer(r[1]).tolist() == x.tolist()
        assert np.frombuffer(r[2]).tolist() == f.tolist()
        assert np.frombuffer(r[3], dtype=np.int64).tolist() == list(duals.keys())
        assert np.frombuffer(r[4]).tolist() == list(duals.values())
