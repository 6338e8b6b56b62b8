"""Small cases of every schedule for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
config-1 geometry (8 frames 64x64, p=2, M=3, 2 levels, n=2) in balanced, accurate and fast mode, a 1-level
p=3 blend (mid kernel), tree build/query with cells, interpolation with alignment and tracking, and the
NNF API with jump flood.  Development aid; see profiles/r01_sanitizer.txt."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_09265_b200 as P
from paper_2311_09265_b200 import shard
from synth import moving_texture

g, s = moving_texture(8, 64, 64, seed=3)
gd, sd = torch.from_numpy(g).cuda(), torch.from_numpy(s).cuda()
ctx = P.Context(0)
for loss, sched in ((P.GUIDE_STYLE, P.DIRECT), (P.MEAN_ALIGN, P.DIRECT), (P.GUIDE_STYLE, P.TREE)):
    ctx.fb_blend_window(P.MatchCfg(iters_per_level=2, loss=loss), sched, gd, sd, 3)
ctx.fb_blend_window(P.MatchCfg(patch_radius=3, levels=1, iters_per_level=1, loss=P.GUIDE_STYLE), P.DIRECT, gd, sd, 2)
cfg = P.MatchCfg(iters_per_level=1, loss=P.GUIDE_STYLE)
plan = shard.plan_shards(8, 3, 2, "tree")
pool = {}
for r in range(2):
    f0, f1 = shard.halo_range(8, 3, *plan[r])
    b = shard.cells_to_build(plan, 8, 3, r)
    if b:
        T, _ = ctx.fb_tree_build_cells(cfg, 8, f0, gd[f0:f1], sd[f0:f1], b)
        pool.update({c: T[k] for k, c in enumerate(b)})
for r in range(2):
    t0, t1 = plan[r]
    f0, f1 = shard.halo_range(8, 3, t0, t1)
    need = shard.tree_cells_needed(8, 3, t0, t1)
    ctx.fb_tree_query(cfg, 8, f0, gd[f0:f1], sd[f0:f1], 3, t0, t1, need, [pool[c] for c in need])
ctx.fb_interpolate_keyframes(P.MatchCfg(iters_per_level=1, loss=P.PAIRWISE, tracking=1), gd, [0, 7], sd[[0, 7]])
ctx.fb_nnf_estimate(P.MatchCfg(iters_per_level=2, loss=P.GUIDE_STYLE, prop_scales=3), gd[:2], gd[2:4], sd[:2])
torch.cuda.synchronize()
print("sanitize case done, launches", ctx.launch_count())
