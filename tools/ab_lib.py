"""A/B of alternative library builds (tools/build_variant.sh): each runs in its own process with FB_LIB set;
prints best-of-reps step time, the top kernel classes and an output hash (bit-identity check).
Development aid, not the bench.  usage: python tools/ab_lib.py N mode lib1.so [lib2.so ...]"""
import hashlib, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, time, hashlib
sys.path.insert(0, ROOT)
import torch
import paper_2311_09265_b200 as P
from synth import moving_texture
N, mode = int(sys.argv[1]), sys.argv[2]
g, s = moving_texture(N, 512, 512)
gd, sd = torch.from_numpy(g).cuda(), torch.from_numpy(s).cuda()
cfg = P.MatchCfg(loss=P.MEAN_ALIGN if mode == "accurate" else P.GUIDE_STYLE)
sched = P.TREE if mode == "fast" else P.DIRECT
M = 30 if mode == "fast" else 15
ctx = P.Context(0)
best = 1e9
for rep in range(3):
    torch.cuda.synchronize(); t = time.time()
    out, st = ctx.fb_blend_window(cfg, sched, gd, sd, M)
    torch.cuda.synchronize(); best = min(best, time.time() - t)
h = hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:12]
ctx.profile_enable(True); ctx.profile_reset()
ctx.fb_blend_window(cfg, sched, gd, sd, M); torch.cuda.synchronize()
prof = ctx.profile_read()
top = sorted(prof.items(), key=lambda kv: -kv[1]["ms"])[:7]
print(f"best {best*1e3:.1f} ms  {st['candidate_evals']/best/1e9:.2f} G evals/s  hash {h}")
print("   ", ", ".join(f"{k} {v['ms']:.1f}" for k, v in top))
'''.replace("ROOT", repr(ROOT))
N, mode = sys.argv[1], sys.argv[2]
for lib in sys.argv[3:]:
    env = dict(os.environ, FB_LIB=os.path.abspath(lib))
    r = subprocess.run([sys.executable, "-c", CHILD, N, mode], env=env, capture_output=True, text=True, timeout=900)
    print(f"== {os.path.basename(lib)}", flush=True)
    print(r.stdout.strip() or r.stderr.strip()[-2000:], flush=True)
