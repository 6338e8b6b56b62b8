"""Per-shard work of the multi-GPU plan, timed on ONE GPU (development aid; no collectives involved).
For world sizes G, each rank's device work (its targets; fast mode: its owned cells, then its queries with
the cells it would receive) is run alone and timed with CUDA events; projected strong-scaling efficiency
= T(1 GPU) / (G * max over ranks), communication excluded (halo frames / cells over NVLink: < 1 ms).
usage: python tools/shard_sim.py mode [N] [G ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_09265_b200 as P
from paper_2311_09265_b200 import shard
from synth import moving_texture

mode = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 200
Gs = [int(x) for x in sys.argv[3:]] or [2, 4, 8]
M = 30 if mode == "fast" else 15
g, s = moving_texture(N, 512, 512)
gd, sd = torch.from_numpy(g).cuda(), torch.from_numpy(s).cuda()
cfg = P.MatchCfg(loss=P.MEAN_ALIGN if mode == "accurate" else P.GUIDE_STYLE)
sched = P.TREE if mode == "fast" else P.DIRECT
recompute = os.environ.get("SIM_RECOMPUTE") == "1"  # fast mode: every shard rebuilds its halo cells instead
ctx = P.Context(0)


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(); r = fn(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1), r


ctx.fb_blend_window(cfg, sched, gd[:min(N, 40)], sd[:min(N, 40)], M)  # warm-up
t1, (ref, _) = timed(lambda: ctx.fb_blend_window(cfg, sched, gd, sd, M))
print(f"{mode} N={N} M={M}: 1 GPU {t1:.0f} ms", flush=True)
for G in Gs:
    plan = shard.plan_shards(N, M, G, "tree" if sched == P.TREE else "direct")
    times, pool, build_ms = [], {}, []
    if sched == P.TREE and not recompute:
        for r in range(G):
            f0, f1 = shard.halo_range(N, M, *plan[r])
            b = shard.cells_to_build(plan, N, M, r)
            ms, res = timed(lambda: ctx.fb_tree_build_cells(cfg, N, f0, gd[f0:f1], sd[f0:f1], b)) if b else (0.0, None)
            if b:
                pool.update({c: res[0][k] for k, c in enumerate(b)})
            build_ms.append(ms)
    ok = True
    for r in range(G):
        t0, tt1 = plan[r]
        f0, f1 = shard.halo_range(N, M, t0, tt1)
        if sched == P.TREE and not recompute:
            need = shard.tree_cells_needed(N, M, t0, tt1)
            ms, (out, _) = timed(lambda: ctx.fb_tree_query(cfg, N, f0, gd[f0:f1], sd[f0:f1], M, t0, tt1, need,
                                                           [pool[c] for c in need]))
            ms += build_ms[r]
        else:
            ms, (out, _) = timed(lambda: ctx.fb_blend_window_range(cfg, sched, N, f0, gd[f0:f1], sd[f0:f1], M, t0, tt1))
        ok &= torch.equal(out, ref[t0:tt1])
        times.append(ms)
    print(f"  G={G}: per-rank ms min {min(times):.0f} max {max(times):.0f}; projected efficiency "
          f"{t1 / (G * max(times)):.3f}; shards bit-identical to the 1-GPU result: {ok}", flush=True)
