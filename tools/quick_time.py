"""Quick timing of config 2 (accurate, 200x512^2, M=15) — development aid, not the bench."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_09265_b200 as P
from synth import moving_texture
N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
mode = sys.argv[2] if len(sys.argv) > 2 else "accurate"
t = time.time(); g, s = moving_texture(N, 512, 512); print("gen", time.time() - t, flush=True)
ctx = P.Context(0)
cfg = P.MatchCfg(loss=P.MEAN_ALIGN if mode == "accurate" else P.GUIDE_STYLE)
sched = P.TREE if mode == "fast" else P.DIRECT
M = 30 if mode == "fast" else 15
gd, sd = torch.from_numpy(g).cuda(), torch.from_numpy(s).cuda()
for rep in range(2):
    torch.cuda.synchronize(); t = time.time()
    out, st = ctx.fb_blend_window(cfg, sched, gd, sd, M)
    torch.cuda.synchronize(); dt = time.time() - t
    print(mode, N, f"{dt:.3f}s", st, f"{st['candidate_evals']/dt/1e9:.2f} Gevals/s", f"{N/dt:.2f} fps", flush=True)
print("ws GB", ctx.ws.numel() / 1e9, "launches", ctx.launch_count())
