"""Full-size parity at BASELINE.json's configurations, in the launch configuration bench.py times, on
sampled output frames the oracle recomputes with their whole dependency closure (targets subset)."""
import numpy as np
import pytest
import torch

import oracle as O
from synth import moving_texture

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

FRAME_TOL = 1.0  # 1/255 on [0,1], in 8-bit units (north_star)


@pytest.fixture(scope="module")
def P():
    import paper_2311_09265_b200 as P
    return P


@pytest.fixture(scope="module")
def ctx(P):
    return P.Context(0)


def ocfg(c):
    return O.Cfg(c.patch_radius, c.levels, c.iters_per_level, c.rs_radius0, c.rs_steps, c.alpha, c.loss, c.init, c.seed,
                 c.prop_scales, c.tracking)


def check(got, ref):
    got = got.detach().cpu().numpy()
    d = np.abs(got.astype(np.float64) - ref.astype(np.float64))
    assert d.max() <= FRAME_TOL, f"max |diff| = {d.max()}"
    assert np.array_equal(got, ref), f"{np.mean(got != ref):.3g} of values differ (max {d.max()})"


@pytest.fixture(scope="module")
def video512():
    return moving_texture(200, 512, 512)


def test_config2_accurate_200x512_window15(P, ctx, video512):
    """configs[1]: accurate mode, 200 x 512^2, patch 5, window 15 (the bench workload)."""
    g, s = video512
    cfg = P.MatchCfg(loss=P.MEAN_ALIGN)
    out, st = ctx.fb_blend_window_range(cfg, P.DIRECT, 200, 0, torch.from_numpy(g).cuda(),
                                        torch.from_numpy(s).cuda(), 15, 0, 200)
    assert st["nnf_pairs"] == 5760 and st["candidate_evals"] == 5760 * 25615360
    targets = [0, 199]
    ref, pairs, _ = O.blend_direct(ocfg(cfg), g, s, 15, targets=targets)
    assert pairs == 30
    check(out[targets], ref)


def test_config3_fast_200x512_window30(P, ctx, video512):
    """configs[2]: fast (tree) mode, 200 x 512^2, window 30."""
    g, s = video512
    cfg = P.MatchCfg(loss=P.GUIDE_STYLE)
    out, st = ctx.fb_blend_window(cfg, P.TREE, torch.from_numpy(g).cuda(), torch.from_numpy(s).cuda(), 30)
    targets = [0, 150]
    ref, _, _ = O.blend_tree(ocfg(cfg), g, s, 30, targets=targets)
    check(out[targets], ref)


@pytest.mark.parametrize("align", [False, True])
def test_config4_interpolation_768(P, ctx, align):
    """configs[3]: 2 keyframes (0 and 101) rendering the 100 in-between 768^2 frames (with and without
    the Eq. 10 alignment of the two NNFs)."""
    g, s = moving_texture(102, 768, 768, seed=4)
    keys = [0, 101]
    cfg = P.MatchCfg(loss=P.PAIRWISE if align else P.GUIDE_STYLE)
    out, st = ctx.fb_interpolate_keyframes(cfg, torch.from_numpy(g).cuda(), keys, torch.from_numpy(s[keys]).cuda())
    assert st["nnf_pairs"] == 200
    targets = [0, 1, 50, 100]
    ref, _, _ = O.interpolate(ocfg(cfg), g, keys, s[keys], targets=targets)
    check(out[targets], ref)


def test_config5_1080p_patch7_window15_shard(P, ctx):
    """configs[4] geometry (1920x1080, patch 7, window 15) through the shard entry point the 8-GPU
    run uses: the shard owning target 0 with its halo of M frames."""
    g, s = moving_texture(16, 1080, 1920, seed=5)
    cfg = P.MatchCfg(patch_radius=3, loss=P.GUIDE_STYLE)
    out, st = ctx.fb_blend_window_range(cfg, P.DIRECT, 1000, 0, torch.from_numpy(g).cuda(), torch.from_numpy(s).cuda(),
                                        15, 0, 1)
    assert st["nnf_pairs"] == 15 and st["candidate_evals"] == 15 * 216537300
    ref, _, _ = O.blend_direct(ocfg(cfg), g, s, 15, targets=[0])
    check(out[0:1], ref)
