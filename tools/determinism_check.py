"""Repeat one blend many times and check every output is bit-identical (race / uninitialised-read check).
usage: python tools/determinism_check.py N mode reps"""
import hashlib, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_09265_b200 as P
from synth import moving_texture
N, mode, reps = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
g, s = moving_texture(N, 512, 512)
gd, sd = torch.from_numpy(g).cuda(), torch.from_numpy(s).cuda()
cfg = P.MatchCfg(loss=P.MEAN_ALIGN if mode == "accurate" else P.GUIDE_STYLE)
sched = P.TREE if mode == "fast" else P.DIRECT
M = 30 if mode == "fast" else 15
hs = {}
for rep in range(reps):
    ctx = P.Context(0) if rep % 3 == 0 else ctx  # fresh context (and workspace) every third rep
    out, st = ctx.fb_blend_window(cfg, sched, gd, sd, M)
    h = hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:12]
    hs.setdefault(h, []).append(rep)
print(mode, N, "distinct outputs:", len(hs), {k: v[:8] for k, v in hs.items()}, flush=True)
