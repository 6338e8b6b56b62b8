"""Timing of one config-5 shard (1920x1080, p=3, M=15, balanced) through fb_blend_window_range:
targets [0, T) of a 1000-frame video from local frames [0, T+M).  Usage: python tools/config5_time.py [T]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_09265_b200 as P  # noqa: E402
from synth import moving_texture  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 8
M = 15
g, s = moving_texture(T + M, 1080, 1920, seed=5)
gd, sd = torch.from_numpy(g).cuda(), torch.from_numpy(s).cuda()
ctx = P.Context(0)
cfg = P.MatchCfg(patch_radius=3, loss=P.GUIDE_STYLE)
ctx.fb_blend_window_range(cfg, P.DIRECT, 1000, 0, gd, sd, M, 0, T)
torch.cuda.synchronize()
ctx.profile_enable(True)
t0 = time.time()
out, st = ctx.fb_blend_window_range(cfg, P.DIRECT, 1000, 0, gd, sd, M, 0, T)
torch.cuda.synchronize()
dt = time.time() - t0
prof = ctx.profile_read()
print(f"config-5 shard: {T} targets, {st['nnf_pairs']} pairs, {dt:.2f} s, {st['candidate_evals'] / dt / 1e9:.2f} G evals/s, "
      f"{dt / st['nnf_pairs'] * 29760 / 8:.1f} s projected per GPU for the 8-GPU run (29760 pairs)")
for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])[:8]:
    print(f"  {k:10s} {v['ms']:9.1f} ms")
