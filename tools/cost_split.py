"""Development aid: per-kernel-class device time of one N-frame 512^2 blend under configuration variants (which
part of a kernel's time is the random search, the propagation, ...).  Not the bench.
usage: python tools/cost_split.py N mode [variant ...]   variant = name:key=val,key=val (MatchCfg fields) or
       name:opt.OPTION=val (fb_set_option)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_09265_b200 as P  # noqa: E402
from synth import moving_texture  # noqa: E402

N, mode = int(sys.argv[1]), sys.argv[2]
variants = sys.argv[3:] or ["default:"]
g, s = moving_texture(N, 512, 512)
gd, sd = torch.from_numpy(g).cuda(), torch.from_numpy(s).cuda()
sched = P.TREE if mode == "fast" else P.DIRECT
M = 30 if mode == "fast" else 15
for v in variants:
    name, _, spec = v.partition(":")
    kw, opts = {}, {}
    for item in filter(None, spec.split(",")):
        k, _, val = item.partition("=")
        if k.startswith("opt."):
            opts[k[4:]] = int(val)
        else:
            kw[k] = float(val) if k == "alpha" else int(val)
    cfg = P.MatchCfg(loss=P.MEAN_ALIGN if mode == "accurate" else P.GUIDE_STYLE, **kw)
    ctx = P.Context(0)
    for k, val in opts.items():
        ctx.set_option(getattr(P.fb, "OPT_" + k), val)
    ctx.fb_blend_window(cfg, sched, gd, sd, M)
    ctx.profile_enable(True)
    ctx.profile_reset()
    out, st = ctx.fb_blend_window(cfg, sched, gd, sd, M)
    torch.cuda.synchronize()
    prof = ctx.profile_read()
    tot = sum(x["ms"] for x in prof.values())
    top = sorted(prof.items(), key=lambda kv: -kv[1]["ms"])[:8]
    print(f"{name:14s} total {tot:7.1f} ms, {st['candidate_evals']/1e9:.2f} G evals | " +
          ", ".join(f"{k} {x['ms']:.1f}" for k, x in top), flush=True)
    del ctx
