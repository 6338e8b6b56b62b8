"""A/B of a context option (fb_set_option, include/fb.h): same inputs, every value, outputs compared bit for bit,
step times and the top kernel classes printed.  Development aid, not the bench.
usage: python tools/ab_env.py OPTION N mode [reps] [v1,v2,...]   (OPTION: FUSED_ITER, FUSE13, PHASE0_MID,
       TGT_REG_ROWS, L1_FAST; values default 0,1)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_09265_b200 as P  # noqa: E402
from synth import moving_texture  # noqa: E402

opt, N, mode = sys.argv[1], int(sys.argv[2]), sys.argv[3]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
values = [int(v) for v in sys.argv[5].split(",")] if len(sys.argv) > 5 else [0, 1]
option = getattr(P.fb, "OPT_" + opt)
g, s = moving_texture(N, 512, 512)
gd, sd = torch.from_numpy(g).cuda(), torch.from_numpy(s).cuda()
cfg = P.MatchCfg(loss=P.MEAN_ALIGN if mode == "accurate" else P.GUIDE_STYLE)
sched = P.TREE if mode == "fast" else P.DIRECT
M = 30 if mode == "fast" else 15
outs = {}
for val in values:
    ctx = P.Context(0)
    ctx.set_option(option, val)
    best = 1e9
    for rep in range(reps):
        torch.cuda.synchronize()
        t = time.time()
        out, st = ctx.fb_blend_window(cfg, sched, gd, sd, M)
        torch.cuda.synchronize()
        best = min(best, time.time() - t)
    outs[val] = out.clone()
    ctx.profile_enable(True)
    ctx.profile_reset()
    ctx.fb_blend_window(cfg, sched, gd, sd, M)
    torch.cuda.synchronize()
    prof = ctx.profile_read()
    ctx.profile_enable(False)
    top = sorted(prof.items(), key=lambda kv: -kv[1]["ms"])[:10]
    print("   ", ", ".join(f"{k} {v['ms']:.1f}" for k, v in top), flush=True)
    print(f"{opt}={val}: {mode} N={N} best {best*1e3:.1f} ms, {st['candidate_evals']/best/1e9:.2f} G evals/s", flush=True)
    del ctx
ref = outs[values[0]]
for val in values[1:]:
    print(f"{opt}={val} bit-identical to {opt}={values[0]}:", torch.equal(outs[val], ref),
          "max diff", float((outs[val] - ref).abs().max()))
