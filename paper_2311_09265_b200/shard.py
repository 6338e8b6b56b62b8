"""Multi-GPU frame sharding with a halo.

One process per GPU.  Output targets are split into contiguous ranges balanced by NNF pair count (not
frame count); rank g owns targets [t0, t1) and needs input frames [t0 - M, t1 + M) clipped to the video.
Each rank holds only its own frames; the halo frames are the one real exchange step of the path and
move with torch.distributed point-to-point ops (NCCL over NVLink on the GPU box, gloo in CPU tests).
After the exchange the shards are independent: each calls fb_blend_window_range on its local frames.
Pair-keyed RNG (D21) makes the result identical for every world size.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def direct_pairs(N: int, M: int, i: int) -> int:
    """NNF pairs of target i under the direct schedule: |W_i| - 1 (D3)."""
    return min(N - 1, i + M) - max(0, i - M)


def tree_pairs(N: int, M: int, i: int) -> int:
    """Approximate per-target NNF cost of the tree schedule: the query walks of both orientations
    (the build cells are shared, so they are charged evenly)."""
    def walk(l, r):
        n, x = 0, r
        while x >= l:
            L = 0
            while (x >> L) & 1 and x - (1 << (L + 1)) + 1 >= l:
                L += 1
            n += 1
            x -= 1 << L
        return n - 1
    v = N - 1 - i
    return walk(max(0, i - M), i) + walk(max(0, v - M), v) + 2


def plan_shards(N: int, M: int, world: int, schedule: str = "direct") -> list[tuple[int, int]]:
    """Contiguous target ranges [t0, t1), one per rank, balanced by pair count.  Every rank gets at
    least one target when N >= world (ranks beyond N get empty ranges)."""
    if world <= 1:
        return [(0, N)]
    cost = [(direct_pairs if schedule == "direct" else tree_pairs)(N, M, i) + 1 for i in range(N)]
    prefix = [0]
    for c in cost:
        prefix.append(prefix[-1] + c)
    total = prefix[-1]
    bounds = [0]
    for g in range(1, world):
        target = total * g / world
        i = min(range(N + 1), key=lambda j: (abs(prefix[j] - target), j))
        lo = bounds[-1] + (1 if N >= world else 0)
        hi = N - (world - g) if N >= world else N
        bounds.append(min(max(i, lo), hi))
    bounds.append(N)
    return [(bounds[g], bounds[g + 1]) for g in range(world)]


def halo_range(N: int, M: int, t0: int, t1: int) -> tuple[int, int]:
    """Input frames [f0, f1) rank needs for targets [t0, t1) (empty for an empty range)."""
    if t1 <= t0:
        return t0, t0
    return max(0, t0 - M), min(N, t1 + M)


def owner_of(plan: list[tuple[int, int]], f: int) -> int:
    for g, (a, b) in enumerate(plan):
        if a <= f < b:
            return g
    raise ValueError(f"frame {f} not owned")


def halo_exchange(owned: list[torch.Tensor], plan: list[tuple[int, int]], N: int, M: int, rank: int,
                  group=None) -> tuple[list[torch.Tensor], int]:
    """owned: tensors [t1-t0, ...] of this rank's frames (same plan for every tensor, e.g. guide and
    style).  Returns the local tensors [f1-f0, ...] (owned frames plus halo) and f0.  Each halo frame
    range is received from its owner in one message per (tensor, peer)."""
    t0, t1 = plan[rank]
    f0, f1 = halo_range(N, M, t0, t1)
    locals_ = []
    for x in owned:
        loc = torch.empty((f1 - f0,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        loc[t0 - f0:t1 - f0].copy_(x)
        locals_.append(loc)
    ops = []
    world = len(plan)
    # receives: for every peer, the intersection of my halo with its owned range
    for g in range(world):
        if g == rank:
            continue
        a, b = plan[g]
        lo, hi = max(a, f0), min(b, f1)
        if lo < hi:
            for loc in locals_:
                ops.append(dist.P2POp(dist.irecv, loc[lo - f0:hi - f0], g, group))
    # sends: for every peer, the intersection of its halo with my owned range
    for g in range(world):
        if g == rank:
            continue
        a, b = plan[g]
        pf0, pf1 = halo_range(N, M, a, b)
        lo, hi = max(t0, pf0), min(t1, pf1)
        if lo < hi:
            for x in owned:
                ops.append(dist.P2POp(dist.isend, x[lo - t0:hi - t0].contiguous(), g, group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    return locals_, f0
