"""f3 measurement: reconstruction quality vs candidate evaluations for unit-step (J=1) and
jump-flood (J>1, D41) propagation.  Pairs of synthetic 512x512 guide frames `gap` frames apart; the
remap of the source guide under the estimated NNF is compared with the target guide (PSNR, interior).
Usage: python tools/jf_convergence.py [gap]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_09265_b200 as P  # noqa: E402
from synth import moving_texture  # noqa: E402

gap = int(sys.argv[1]) if len(sys.argv) > 1 else 8
g, _ = moving_texture(64, 512, 512)
pairs = [(i, i + gap) for i in range(0, 64 - gap, 4)]
sg = torch.from_numpy(np.stack([g[a] for a, _ in pairs])).cuda()
tg = torch.from_numpy(np.stack([g[b] for _, b in pairs])).cuda()
keys = [(a, b, 6) for a, b in pairs]
ctx = P.Context(0)
m = 2 + 5
print(f"{len(pairs)} pairs, gap {gap} frames, 512x512, p=2, auto levels")
print(f"{'J':>3s} {'n':>3s} {'evals/pair':>12s} {'PSNR dB':>8s}")
for J in (1, 2, 4):
    for n in (1, 2, 3, 5):
        cfg = P.MatchCfg(iters_per_level=n, loss=P.GUIDE_STYLE, prop_scales=J)
        F, E, X, st = ctx.fb_nnf_estimate(cfg, sg, tg, sg, pair_keys=keys)
        d = (X - tg.float())[:, m:-m, m:-m]
        mse = (d.double() ** 2).mean().item()
        print(f"{J:3d} {n:3d} {st['candidate_evals'] // len(pairs):12d} {10 * np.log10(255.0 ** 2 / mse):8.3f}")
