"""Multi-GPU frame sharding with a halo.

One process per GPU.  Output targets are split into contiguous ranges balanced by NNF pair count (not
frame count); rank g owns targets [t0, t1) and needs input frames [t0 - M, t1 + M) clipped to the video.
Each rank holds only its own frames; the halo frames are the one real exchange step of the path and
move with torch.distributed point-to-point ops (NCCL over NVLink on the GPU box; gloo -- host-staged for
device tensors -- in the CPU tests and the world-2-on-one-GPU correctness runs).  Reading D43:
the exchange transport is torch.distributed, not an fb_group inside the C ABI.
After the exchange the shards are independent: each calls fb_blend_window_range on its local frames.
Pair-keyed RNG (D21) makes the result identical for every world size.
"""
from __future__ import annotations

import contextlib

import torch
import torch.distributed as dist


@contextlib.contextmanager
def _nvtx(name: str):
    """NVTX range around an exchange step (no-op without CUDA, e.g. in the gloo CPU tests)."""
    if torch.cuda.is_available():
        torch.cuda.nvtx.range_push(name)
        try:
            yield
        finally:
            torch.cuda.nvtx.range_pop()
    else:
        yield


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
    return plan_by_cost([(direct_pairs if schedule == "direct" else tree_pairs)(N, M, i) + 1 for i in range(N)], world)


def plan_by_cost(cost: list[int], world: int) -> list[tuple[int, int]]:
    """Contiguous ranges of len(cost) items, one per rank, with near-equal cost sums."""
    N = len(cost)
    if world <= 1:
        return [(0, N)]
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


def _host_staged(group=None) -> bool:
    """gloo moves CPU tensors only: device tensors are staged through host memory (the world-2-on-one-GPU
    correctness runs; on the 8-GPU box the backend is NCCL and tensors move device to device)."""
    return dist.get_backend(group) == "gloo"


def _p2p(ops: list, group=None):
    """batch_isend_irecv of (op, tensor, peer) triples; with host staging, device tensors are copied to pinned
    host buffers for the transfer and received ones copied back."""
    if not ops:
        return
    staged = _host_staged(group)
    real, back = [], []
    for op, t, peer in ops:
        if staged and t.is_cuda:
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            if op is dist.isend:
                h.copy_(t)
            else:
                back.append((t, h))
            t = h
        real.append(dist.P2POp(op, t, _global(peer, group), group))
    for r in dist.batch_isend_irecv(real):
        r.wait()
    for t, h in back:
        t.copy_(h, non_blocking=True)


def _global(g: int, group=None) -> int:
    """Plan index (rank within `group`) -> global rank, as torch.distributed's P2P and broadcast expect."""
    return g if group is None else dist.get_global_rank(group, g)


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
                ops.append((dist.irecv, loc[lo - f0:hi - f0], g))
    # sends: for every peer, the intersection of its halo with my owned range
    for g in range(world):
        if g == rank:
            continue
        a, b = plan[g]
        pf0, pf1 = halo_range(N, M, a, b)
        lo, hi = max(t0, pf0), min(t1, pf1)
        if lo < hi:
            for x in owned:
                ops.append((dist.isend, x[lo - t0:hi - t0].contiguous(), g))
    with _nvtx("halo exchange"):
        _p2p(ops, group)
    return locals_, f0


def blend_direct_sharded(ctx, cfg, plan: list[tuple[int, int]], N: int, M: int, rank: int, guide_own, style_own,
                         out=None, group=None):
    """Direct schedule (balanced / accurate) of this rank's targets: halo exchange, then fb_blend_window_range
    on the local frames.  A rank with an empty range takes part in the exchange and returns (None, {})."""
    t0, t1 = plan[rank]
    (g_loc, s_loc), f0 = halo_exchange([guide_own, style_own], plan, N, M, rank, group)
    if t1 <= t0:
        return None, {}
    from .fb import DIRECT
    return ctx.fb_blend_window_range(cfg, DIRECT, N, f0, g_loc, s_loc, M, t0, t1, out=out)


# ---------------------------------------------------------------------------------------------- tree
# Tree schedule (Alg. 3-5): a shard's Alg. 5 queries visit blending-table cells BT(node, L) of nodes up to
# M frames outside its targets.  Rebuilding them (fb_blend_window_range) costs ~20 % extra NNFs per GPU at
# G = 8; instead every cell has one owner (the rank owning the node's frame), owners build the
# cells any rank needs, and the cells move point-to-point once, before the queries (include/fb.h).

def query_nodes(l: int, r: int) -> list[tuple[int, int]]:
    """Alg. 5's walk over [l, r] (D23: i <- i - 2^L): the (node, L) pairs it visits."""
    out, i = [], r
    while i >= l:
        L = 0
        while (i >> L) & 1 and i - (1 << (L + 1)) + 1 >= l:
            L += 1
        out.append((i, L))
        i -= 1 << L
    return out


def tree_cells_needed(N: int, M: int, t0: int, t1: int) -> list[tuple[int, int, int]]:
    """Cells (orient, node, L >= 1) the queries of targets [t0, t1) visit, in a canonical order."""
    need = set()
    for o in (0, 1):
        for i in range(t0, t1):
            v = i if o == 0 else N - 1 - i
            for node, L in query_nodes(max(0, v - M), v):
                if L >= 1:
                    need.add((o, node, L))
    return sorted(need)


def cell_frame(N: int, cell: tuple[int, int, int]) -> int:
    """Original frame id of a cell's node (its owner is the rank owning that frame)."""
    o, j, _ = cell
    return j if o == 0 else N - 1 - j


def exchange_cells(plan: list[tuple[int, int]], N: int, M: int, rank: int, built: dict, texels: int,
                   device, group=None) -> dict:
    """built: {cell: tensor [texels, 4]} of the cells this rank owns and some rank needs.  Sends each peer
    the cells it needs from this rank (one message per peer, cells in canonical order) and receives the
    cells this rank needs from their owners.  Returns {cell: tensor} for every cell this rank's queries
    visit (its own built ones plus the received ones)."""
    world = len(plan)
    t0, t1 = plan[rank]
    mine = tree_cells_needed(N, M, t0, t1) if t1 > t0 else []
    owner = {c: owner_of(plan, cell_frame(N, c)) for c in mine}
    ops, recv = [], {}
    for g in range(world):
        if g == rank:
            continue
        a, b = plan[g]
        theirs = [c for c in tree_cells_needed(N, M, a, b) if owner_of(plan, cell_frame(N, c)) == rank] if b > a else []
        if theirs:
            ops.append((dist.isend, torch.stack([built[c] for c in theirs]).contiguous(), g))
        from_g = [c for c in mine if owner[c] == g]
        if from_g:
            buf = torch.empty((len(from_g), texels, 4), dtype=torch.float32, device=device)
            ops.append((dist.irecv, buf, g))
            recv[g] = (from_g, buf)
    with _nvtx("tree cell exchange"):
        _p2p(ops, group)
    cells = {c: built[c] for c in mine if owner[c] == rank}
    for from_g, buf in recv.values():
        for k, c in enumerate(from_g):
            cells[c] = buf[k]
    return cells


def cells_to_build(plan: list[tuple[int, int]], N: int, M: int, rank: int) -> list[tuple[int, int, int]]:
    """Cells this rank owns that some rank's queries visit (canonical order)."""
    need = set()
    for a, b in plan:
        if b > a:
            need.update(tree_cells_needed(N, M, a, b))
    return sorted(c for c in need if owner_of(plan, cell_frame(N, c)) == rank)


def blend_tree_exchange(ctx, cfg, plan: list[tuple[int, int]], N: int, M: int, rank: int, guide_loc, style_loc,
                        f0: int, out=None, group=None):
    """Fast-mode blend of this rank's targets with cell exchange: build owned cells, exchange, query."""
    t0, t1 = plan[rank]
    H, W = int(guide_loc.shape[1]), int(guide_loc.shape[2])
    texels = ctx.tree_cell_texels(cfg, H, W)
    build = cells_to_build(plan, N, M, rank)
    built, st_b = {}, {}
    if build:
        T, st_b = ctx.fb_tree_build_cells(cfg, N, f0, guide_loc, style_loc, build)
        built = {c: T[k] for k, c in enumerate(build)}
    cells = exchange_cells(plan, N, M, rank, built, texels, guide_loc.device, group)
    if t1 <= t0:  # an empty range builds and sends nothing, and has no queries
        return None, st_b
    order = sorted(cells)
    out, st_q = ctx.fb_tree_query(cfg, N, f0, guide_loc, style_loc, M, t0, t1, order, [cells[c] for c in order],
                                  out=out)
    return out, {k: st_q.get(k, 0) + st_b.get(k, 0) for k in st_q}


# ---------------------------------------------------------------------------------------- interpolation
# Eq. 9: every frame's NNFs read only its own guide frame and the keyframes, so the frames
# shard with no data-path exchange beyond the keyframes themselves, which are broadcast once: the key
# styles from the rank that holds them (rank 0), each key's guide frame from the rank owning that frame.

def interp_pairs(N: int, keys: list[int], m: int) -> int:
    """NNF pairs of frame m: 0 for a keyframe, else the number of keys on its sides (1 or 2)."""
    if m in keys:
        return 0
    return int(any(k < m for k in keys)) + int(any(k > m for k in keys))


def plan_interp_shards(N: int, keys: list[int], world: int) -> list[tuple[int, int]]:
    return plan_by_cost([interp_pairs(N, keys, m) + 1 for m in range(N)], world)


def broadcast_keyframes(plan: list[tuple[int, int]], keys: list[int], rank: int, guide_own: torch.Tensor,
                        key_style: torch.Tensor | None, group=None) -> tuple[torch.Tensor, torch.Tensor]:
    """Returns (key_guide [K,H,W,3], key_style [K,H,W,3]) on every rank: key styles broadcast from rank 0
    (key_style is read there only), each key's guide frame from the rank owning that frame."""
    with _nvtx("keyframe broadcast"):
        return _broadcast_keyframes(plan, keys, rank, guide_own, key_style, group)


def _broadcast_keyframes(plan, keys, rank, guide_own, key_style, group):
    t0, _ = plan[rank]
    shape = tuple(guide_own.shape[1:])
    K = len(keys)
    kg = torch.empty((K,) + shape, dtype=guide_own.dtype, device=guide_own.device)
    for k, f in enumerate(keys):
        src = owner_of(plan, f)
        if src == rank:
            kg[k].copy_(guide_own[f - t0])
        _broadcast(kg[k], src, group)
    ks = key_style.contiguous() if rank == 0 else torch.empty((K,) + shape, dtype=guide_own.dtype,
                                                              device=guide_own.device)
    _broadcast(ks, 0, group)
    return kg, ks


def _broadcast(t: torch.Tensor, src: int, group=None):
    """dist.broadcast from plan index `src` (host-staged under gloo, like _p2p)."""
    if _host_staged(group) and t.is_cuda:
        h = t.cpu()
        dist.broadcast(h, _global(src, group), group)
        t.copy_(h)
    else:
        dist.broadcast(t, _global(src, group), group)


def interpolate_sharded(ctx, cfg, plan: list[tuple[int, int]], N: int, keys: list[int], rank: int,
                        guide_own: torch.Tensor, key_style: torch.Tensor | None, out=None, group=None):
    """This rank's frames [t0, t1) of the keyframe interpolation (fb_interpolate_keyframes_range)."""
    t0, t1 = plan[rank]
    kg, ks = broadcast_keyframes(plan, keys, rank, guide_own, key_style, group)
    if t1 <= t0:
        return None, {}
    return ctx.fb_interpolate_keyframes_range(cfg, N, t0, t1, guide_own, keys, kg, ks, out=out)
