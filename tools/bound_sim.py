"""Development aid (not the product, not a test): how many random-search candidates a cheap lower bound of
the patch loss would reject before any patch row is gathered, against the first-row partial-distance test.

Runs the oracle on one accurate-mode-shaped pair to get a converged (F, E, X), then draws random-search
candidates around F at every radius of the schedule and, per candidate, compares
  full   = the Eq. 3 loss (float64),
  row0   = its first patch row (the current elimination test after one row),
  mean   = Cauchy-Schwarz on patch sums: sum_c (sum_i a_ic - sum_i b_ic)^2 / n  <=  sum_ic (a_ic - b_ic)^2,
  rows   = the same per patch row (5 row sums per channel).
usage: python tools/bound_sim.py [H] [pair_distance]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from synth import moving_texture  # noqa: E402

H = int(sys.argv[1]) if len(sys.argv) > 1 else 192
dj = int(sys.argv[2]) if len(sys.argv) > 2 else 4
p, alpha = 2, 10.0
g, s = moving_texture(dj + 1, H, H)
frames = np.concatenate([g[[dj, 0]], s[[dj]]]).astype(np.float32)
tasks = [dict(src_guide=0, tgt_guide=1, src_style=2, src_id=dj, tgt_id=0, tag=0)]
cfg = O.Cfg(iters_per_level=5, loss=O.GUIDE_STYLE)
F, E, X, _ = O.nnf(cfg, frames, tasks)
F, E, X = F[0], E[0].astype(np.float64), X[0].astype(np.float64)
G_s, S_s, G_t = (frames[i].astype(np.float64) for i in (0, 2, 1))
T_aux = X  # the style target of the last refresh (S-hat)
D = 2 * p + 1
n = D * D


def pad(a):
    return np.pad(a, ((p, p), (p, p), (0, 0)))


Gs, Ss, Gt, Tt = pad(G_s), pad(S_s), pad(G_t), pad(T_aux)


def patches(A, r, c):  # [..., D, D, 3] patches centred at (r, c) of an unpadded-coordinate grid
    rr = r[..., None, None] + np.arange(D)[:, None]
    cc = c[..., None, None] + np.arange(D)[None, :]
    return A[rr, cc]


rows, cols = np.meshgrid(np.arange(H), np.arange(H), indexing="ij")
tg, ta = patches(Gt, rows, cols), patches(Tt, rows, cols)
rng = np.random.default_rng(0)
R = H
tot = dict(cands=0, lose=0, row0=0, mean=0, rows=0, mean_or_row0=0)
print(f"H={H}, pair distance {dj}: median E {np.median(E):.0f}")
while R >= 1:
    off = rng.integers(-R, R + 1, size=(H, H, 2))
    cr = np.clip(F[..., 0] + off[..., 0], 0, H - 1)
    cc = np.clip(F[..., 1] + off[..., 1], 0, H - 1)
    sg, ss = patches(Gs, cr, cc), patches(Ss, cr, cc)
    dg, ds = (sg - tg) ** 2, (ss - ta) ** 2
    full = alpha * dg.sum((-3, -2, -1)) + ds.sum((-3, -2, -1))
    row0 = alpha * dg[..., 0, :, :].sum((-2, -1)) + ds[..., 0, :, :].sum((-2, -1))
    mean = (alpha * ((sg.sum((-3, -2)) - tg.sum((-3, -2))) ** 2).sum(-1)
            + ((ss.sum((-3, -2)) - ta.sum((-3, -2))) ** 2).sum(-1)) / n
    rws = (alpha * ((sg.sum(-2) - tg.sum(-2)) ** 2).sum((-2, -1))
           + ((ss.sum(-2) - ta.sum(-2)) ** 2).sum((-2, -1))) / D
    lose = full >= E
    st = dict(cands=lose.size, lose=lose.sum(), row0=(row0 >= E).sum(), mean=(mean >= E).sum(),
              rows=(rws >= E).sum(), mean_or_row0=((mean >= E) | (row0 >= E)).sum())
    for k in tot:
        tot[k] += st[k]
    print(f"R={R:4d}: lose {st['lose']/st['cands']:.3f}  rejected by row0 {st['row0']/st['cands']:.3f}  "
          f"mean {st['mean']/st['cands']:.3f}  row sums {st['rows']/st['cands']:.3f}  "
          f"mean|row0 {st['mean_or_row0']/st['cands']:.3f}")
    R >>= 1
c = tot["cands"]
print("all radii: " + "  ".join(f"{k} {v/c:.3f}" for k, v in tot.items() if k != "cands"))

# variants of the bound with compact sums (8-byte texels): guide-only, and style sums quantised to 32-unit bins
tot2 = dict(cands=0, lose=0, full_mean=0, guide_only=0, qstyle=0)
R = H
rng = np.random.default_rng(1)
while R >= 1:
    off = rng.integers(-R, R + 1, size=(H, H, 2))
    cr = np.clip(F[..., 0] + off[..., 0], 0, H - 1)
    cc = np.clip(F[..., 1] + off[..., 1], 0, H - 1)
    sg, ss = patches(Gs, cr, cc), patches(Ss, cr, cc)
    full = alpha * ((sg - tg) ** 2).sum((-3, -2, -1)) + ((ss - ta) ** 2).sum((-3, -2, -1))
    gl = alpha * ((sg.sum((-3, -2)) - tg.sum((-3, -2))) ** 2).sum(-1) / n
    ssum, tsum = ss.sum((-3, -2)), ta.sum((-3, -2))
    sl = ((ssum - tsum) ** 2).sum(-1) / n
    q = np.floor(ssum / 32) * 32
    dq = np.maximum(np.maximum(q - tsum, tsum - (q + 31)), 0)
    ql = (dq ** 2).sum(-1) / n
    for k, v in (("cands", full.size), ("lose", (full >= E).sum()), ("full_mean", (gl + sl >= E).sum()),
                 ("guide_only", (gl >= E).sum()), ("qstyle", (gl + ql >= E).sum())):
        tot2[k] += v
    R >>= 1
print("compact sums: " + "  ".join(f"{k} {v / tot2['cands']:.3f}" for k, v in tot2.items() if k != "cands"))

# partial rows + Cauchy-Schwarz on the remaining rows, for candidates that survive the patch-mean bound
tot3 = dict(surv=0, r0=0, r1=0, r2=0, pde0=0, pde2=0)
R = H
rng = np.random.default_rng(2)
while R >= 1:
    off = rng.integers(-R, R + 1, size=(H, H, 2))
    cr = np.clip(F[..., 0] + off[..., 0], 0, H - 1)
    cc = np.clip(F[..., 1] + off[..., 1], 0, H - 1)
    sg, ss = patches(Gs, cr, cc), patches(Ss, cr, cc)
    dg, ds = alpha * (sg - tg) ** 2, (ss - ta) ** 2
    mean = (alpha * ((sg.sum((-3, -2)) - tg.sum((-3, -2))) ** 2).sum(-1)
            + ((ss.sum((-3, -2)) - ta.sum((-3, -2))) ** 2).sum(-1)) / n
    surv = mean < E
    tot3["surv"] += surv.sum()
    for r_, key in ((0, "r0"), (1, "r1"), (2, "r2")):
        part = dg[..., : r_ + 1, :, :].sum((-3, -2, -1)) + ds[..., : r_ + 1, :, :].sum((-3, -2, -1))
        m = (D - r_ - 1) * D
        rest = (alpha * ((sg[..., r_ + 1:, :, :].sum((-3, -2)) - tg[..., r_ + 1:, :, :].sum((-3, -2))) ** 2).sum(-1)
                + ((ss[..., r_ + 1:, :, :].sum((-3, -2)) - ta[..., r_ + 1:, :, :].sum((-3, -2))) ** 2).sum(-1)) / m
        tot3[key] += (surv & (part + rest >= E)).sum()
        if r_ in (0, 2):
            tot3["pde" + str(r_)] += (surv & (part >= E)).sum()
    R >>= 1
print("among mean-bound survivors: " + "  ".join(f"{k} {v / tot3['surv']:.3f}" for k, v in tot3.items() if k != "surv"))
