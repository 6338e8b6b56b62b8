"""Profiling case for ncu: one accurate-mode blend (config-2 geometry, fewer frames) after a warm-up.
Usage: python tools/prof_case.py [N frames] [mode]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_09265_b200 as P  # noqa: E402
from synth import moving_texture  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 24
mode = sys.argv[2] if len(sys.argv) > 2 else "accurate"
g, s = moving_texture(N, 512, 512)
ctx = P.Context(0)
cfg = P.MatchCfg(loss=P.MEAN_ALIGN if mode == "accurate" else P.GUIDE_STYLE)
sched = P.TREE if mode == "fast" else P.DIRECT
M = 30 if mode == "fast" else 15
gd, sd = torch.from_numpy(g).cuda(), torch.from_numpy(s).cuda()
reps = int(os.environ.get("PROF_REPS", "1"))
for _ in range(reps):
    out, st = ctx.fb_blend_window(cfg, sched, gd, sd, M)
torch.cuda.synchronize()
print(st, "launches", ctx.launch_count())
