"""Per-kernel-class device times (CUDA events via fb_profile_*) of one blend — development aid.
Usage: python tools/kernel_times.py [N] [mode] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_09265_b200 as P  # noqa: E402
from synth import moving_texture  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 48
mode = sys.argv[2] if len(sys.argv) > 2 else "accurate"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
g, s = moving_texture(N, 512, 512)
ctx = P.Context(0)
cfg = P.MatchCfg(loss=P.MEAN_ALIGN if mode == "accurate" else P.GUIDE_STYLE)
sched = P.TREE if mode == "fast" else P.DIRECT
M = 30 if mode == "fast" else 15
gd, sd = torch.from_numpy(g).cuda(), torch.from_numpy(s).cuda()
ctx.fb_blend_window(cfg, sched, gd, sd, M)
torch.cuda.synchronize()
ctx.profile_enable(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    out, st = ctx.fb_blend_window(cfg, sched, gd, sd, M)
e1.record()
torch.cuda.synchronize()
prof = ctx.profile_read()
tot = e0.elapsed_time(e1) / reps
print(f"{mode} N={N}: {tot:.1f} ms/step, {st['candidate_evals'] / tot / 1e6:.2f} G evals/s")
ks = sum(v["ms"] for v in prof.values()) / reps
for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
    ms = v["ms"] / reps
    extra = f"  {v['work'] / (v['ms'] / 1e3) / 1e9:7.2f} G/s" if k.startswith("field") else ""
    print(f"  {k:10s} {v['launches'] // reps:5d} launches {ms:9.2f} ms {ms / ks:6.1%}{extra}")
