"""Multi-GPU host logic on CPU: the pair-balanced shard plan and the halo exchange (gloo, world 2-3)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2311_09265_b200 import shard


def direct_cost(N, M, a, b):
    return sum(shard.direct_pairs(N, M, i) for i in range(a, b))


@pytest.mark.parametrize("N,M,world", [(200, 15, 1), (200, 15, 2), (200, 15, 8), (1000, 15, 8), (200, 30, 8),
                                       (7, 3, 8), (9, 0, 4), (1, 5, 2)])
def test_plan_is_contiguous_covering_and_balanced(N, M, world):
    plan = shard.plan_shards(N, M, world)
    assert len(plan) == world
    assert plan[0][0] == 0 and plan[-1][1] == N
    for (a, b), (c, d) in zip(plan, plan[1:]):
        assert b == c and a <= b
    if N >= world:
        assert all(b > a for a, b in plan)
    if N >= 8 * world and M > 0:
        costs = [direct_cost(N, M, a, b) for a, b in plan]
        assert min(costs) / max(costs) >= 0.9, costs


def test_halo_ranges_cover_every_window():
    N, M = 50, 7
    plan = shard.plan_shards(N, M, 4)
    for t0, t1 in plan:
        f0, f1 = shard.halo_range(N, M, t0, t1)
        for i in range(t0, t1):
            assert f0 <= max(0, i - M) and min(N, i + M + 1) <= f1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, N, M, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)
        full_g = torch.from_numpy(rng.integers(0, 256, size=(N, 6, 7, 3), dtype=np.uint8))
        full_s = torch.from_numpy(rng.integers(0, 256, size=(N, 6, 7, 3), dtype=np.uint8))
        plan = shard.plan_shards(N, M, world)
        t0, t1 = plan[rank]
        (g_loc, s_loc), f0 = shard.halo_exchange([full_g[t0:t1].clone(), full_s[t0:t1].clone()], plan, N, M, rank)
        f1 = f0 + g_loc.shape[0]
        ok = (f0, f1) == shard.halo_range(N, M, t0, t1) and torch.equal(g_loc, full_g[f0:f1]) and \
            torch.equal(s_loc, full_s[f0:f1])
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,N,M", [(2, 20, 3), (3, 12, 6), (2, 5, 9)])
def test_halo_exchange_gloo(world, N, M):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, N, M, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = dict(q.get(timeout=5) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert all(res[r] for r in range(world)), res


# ------------------------------------------------------------------------------ tree cell exchange
def _brute_query_nodes(l, r):
    """Alg. 5 written out (D23): from i = r, take the largest aligned block [i-2^L+1, i] inside [l, r]."""
    out, i = [], r
    while i >= l:
        L = 0
        while (i + 1) % (1 << (L + 1)) == 0 and i - (1 << (L + 1)) + 1 >= l:
            L += 1
        out.append((i, L))
        i -= 1 << L
    return out


@pytest.mark.parametrize("N,M", [(200, 30), (50, 7), (9, 0), (16, 15)])
def test_query_walk_partitions_window(N, M):
    for v in range(N):
        l = max(0, v - M)
        walk = shard.query_nodes(l, v)
        assert walk == _brute_query_nodes(l, v)
        covered = sorted(x for node, L in walk for x in range(node - (1 << L) + 1, node + 1))
        assert covered == list(range(l, v + 1))


@pytest.mark.parametrize("N,M,world", [(200, 30, 8), (200, 30, 3), (50, 7, 4), (12, 6, 3), (5, 9, 2), (7, 3, 8)])
def test_tree_cells_built_once_and_cover_every_need(N, M, world):
    """Across ranks the owned builds partition the cells the whole video's queries visit (no cell is built
    twice, none is missing), and every cell a rank builds reads only frames in its halo range."""
    plan = shard.plan_shards(N, M, world, "tree")
    builds = [shard.cells_to_build(plan, N, M, r) for r in range(world)]
    flat = [c for b in builds for c in b]
    assert len(flat) == len(set(flat))
    assert set(flat) == set(shard.tree_cells_needed(N, M, 0, N))
    for r, b in enumerate(builds):
        f0, f1 = shard.halo_range(N, M, *plan[r])
        for o, j, L in b:
            lo, hi = (j - (1 << L) + 1, j) if o == 0 else (N - 1 - j, N - 1 - j + (1 << L) - 1)
            assert f0 <= lo and hi < f1


def _cell_value(c, texels):
    o, j, L = c
    return torch.full((texels, 4), float(o * 100000 + j * 100 + L))


def _tree_worker(rank, world, port, N, M, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        texels = 5
        plan = shard.plan_shards(N, M, world, "tree")
        built = {c: _cell_value(c, texels) for c in shard.cells_to_build(plan, N, M, rank)}
        got = shard.exchange_cells(plan, N, M, rank, built, texels, torch.device("cpu"))
        t0, t1 = plan[rank]
        need = shard.tree_cells_needed(N, M, t0, t1) if t1 > t0 else []
        ok = sorted(got) == need and all(torch.equal(got[c], _cell_value(c, texels)) for c in need)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,N,M", [(2, 24, 7), (3, 40, 12), (3, 10, 9)])
def test_tree_cell_exchange_gloo(world, N, M):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tree_worker, args=(r, world, port, N, M, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = dict(q.get(timeout=5) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert all(res[r] for r in range(world)), res


# ------------------------------------------------------------------------------ interpolation sharding
@pytest.mark.parametrize("N,keys,world", [(102, [0, 101], 8), (10, [0, 4, 9], 3), (7, [3], 2), (5, [0, 4], 8)])
def test_interp_plan_covers_and_balances(N, keys, world):
    plan = shard.plan_interp_shards(N, keys, world)
    assert plan[0][0] == 0 and plan[-1][1] == N
    for (a, b), (c, d) in zip(plan, plan[1:]):
        assert b == c and a <= b
    if N >= 8 * world:
        costs = [sum(shard.interp_pairs(N, keys, m) + 1 for m in range(a, b)) for a, b in plan]
        assert min(costs) / max(costs) >= 0.85, costs


def _interp_worker(rank, world, port, N, keys, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(9)
        full_g = torch.from_numpy(rng.integers(0, 256, size=(N, 4, 5, 3), dtype=np.uint8))
        full_ks = torch.from_numpy(rng.integers(0, 256, size=(len(keys), 4, 5, 3), dtype=np.uint8))
        plan = shard.plan_interp_shards(N, keys, world)
        t0, t1 = plan[rank]
        kg, ks = shard.broadcast_keyframes(plan, keys, rank, full_g[t0:t1].clone(),
                                           full_ks.clone() if rank == 0 else None)
        ok = torch.equal(kg, full_g[keys]) and torch.equal(ks, full_ks)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,N,keys", [(2, 12, [0, 11]), (3, 15, [0, 7, 14])])
def test_keyframe_broadcast_gloo(world, N, keys):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_interp_worker, args=(r, world, port, N, keys, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = dict(q.get(timeout=5) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert all(res[r] for r in range(world)), res
