"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star): NNF identical on >= 99.9 % of pixels (bit-exact where untied);
patch error relative difference <= 1e-5; output frames max |diff| <= 1/255 on [0,1] (= 1.0 in the
8-bit units of the boundary).  The arithmetic contract makes both sides bit-identical,
so every test also reports the exact-match fraction and most assert it.
"""
import numpy as np
import pytest
import torch

import oracle as O
from synth import constant_video, iid_frames, moving_texture, static_textured_video, textured_frame

pytestmark = pytest.mark.gpu

FRAME_TOL = 1.0  # 1/255 on [0,1] RGB, in 8-bit units


@pytest.fixture(scope="module")
def fb():
    import paper_2311_09265_b200 as P
    return P


@pytest.fixture(scope="module")
def ctx(fb):
    return fb.Context(0)


def ocfg(c):
    return O.Cfg(c.patch_radius, c.levels, c.iters_per_level, c.rs_radius0, c.rs_steps, c.alpha, c.loss, c.init, c.seed,
                 c.prop_scales, c.tracking)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def assert_frames(got, ref, exact=True):
    got = got.detach().cpu().numpy() if torch.is_tensor(got) else got
    d = np.abs(got.astype(np.float64) - ref.astype(np.float64))
    assert d.max() <= FRAME_TOL, f"max |diff| = {d.max()}"
    if exact:
        assert np.array_equal(got, ref), f"not bit-exact: {np.mean(got != ref):.3g} of values differ, max {d.max()}"


def assert_nnf(F, E, Fr, Er, exact=True):
    F = F.cpu().numpy()
    same = np.all(F == Fr, -1)
    assert same.mean() >= 0.999, f"NNF identical on {same.mean():.5f}"
    if E is not None:
        E = E.cpu().numpy()
        rel = np.abs(E.astype(np.float64) - Er) / np.maximum(np.abs(Er.astype(np.float64)), 1e-30)
        assert rel[same].max(initial=0) <= 1e-5
    if exact:
        assert same.all()
        if E is not None:
            assert np.array_equal(E, Er)


# ------------------------------------------------------------------------------ a1 pyramid
@pytest.mark.parametrize("H,W,levels", [(64, 64, 2), (37, 45, 3), (512, 512, 5), (33, 70, 1)])
def test_pyramid_bit_exact(ctx, H, W, levels):
    fr = iid_frames(3, H, W, seed=H)
    got = ctx.fb_build_pyramid(dev(fr), levels).cpu().numpy()
    for b in range(3):
        ref = O.pyramid(fr[b].astype(np.float32), levels)
        off = 0
        for k in range(levels):
            n = (H >> k) * (W >> k)
            lev = got[b, off:off + n].reshape(H >> k, W >> k, 4)
            np.testing.assert_array_equal(lev[..., :3], ref[k])
            assert np.all(lev[..., 3] == 0)
            off += n


# ------------------------------------------------------------------------------ a8 remap
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_remap_bit_exact(ctx, p):
    rng = np.random.default_rng(p)
    B, H, W = 3, 29, 67
    S = (rng.random((B, H, W, 3)) * 255).astype(np.float32)
    F = np.stack([rng.integers(0, H, (B, H, W)), rng.integers(0, W, (B, H, W))], -1).astype(np.int32)
    got = ctx.fb_remap(dev(S), dev(F), p).cpu().numpy()
    for b in range(B):
        np.testing.assert_array_equal(got[b], O.remap(S[b], F[b], p))


# ------------------------------------------------------------------------------ a2-a7 NNF estimation
def _nnf_case(fb, loss, H, W, B=3, seed=4, **kw):
    g, s = moving_texture(B + 1, H, W, seed=seed)
    cfg = fb.MatchCfg(patch_radius=kw.pop("p", 2), iters_per_level=kw.pop("n", 2), loss=loss, **kw)
    sg, tg = g[1:], np.repeat(g[:1], B, 0)
    ss, ts = s[1:], np.repeat(s[:1], B, 0)
    keys = [(j + 1, 0, 6) for j in range(B)]
    frames = np.concatenate([g, s]).astype(np.float32)
    tasks = [dict(src_guide=j + 1, tgt_guide=0, src_style=B + 1 + j + 1, tgt_style=B + 1, group=0, src_id=j + 1,
                  tgt_id=0, tag=6) for j in range(B)]
    if loss != fb.MEAN_ALIGN:
        for t in tasks:
            t["group"] = tasks.index(t)
    if loss == fb.BASE:
        for t in tasks:
            t["src_style"] = -1
    return cfg, (sg, tg, ss, ts, keys), frames, tasks


@pytest.mark.parametrize("loss", [0, 1, 2])
@pytest.mark.parametrize("H,W", [(64, 64), (45, 77)])
def test_nnf_estimate_matches_oracle(fb, ctx, loss, H, W):
    cfg, (sg, tg, ss, ts, keys), frames, tasks = _nnf_case(fb, loss, H, W)
    group = [0] * len(keys) if loss == fb.MEAN_ALIGN else None
    F, E, X, st = ctx.fb_nnf_estimate(cfg, dev(sg), dev(tg), None if loss == 0 else dev(ss),
                                      dev(ts) if loss == 2 else None, group=group, pair_keys=keys)
    Fr, Er, Xr, ev = O.nnf(ocfg(cfg), frames, tasks, want_x=loss != 0)
    assert st["candidate_evals"] == ev and st["nnf_pairs"] == len(keys)
    assert_nnf(F, E, Fr, Er)
    if loss != 0:
        assert_frames(X, Xr)


@pytest.mark.parametrize("kw", [dict(p=1), dict(p=3), dict(p=4, n=1), dict(init=1), dict(rs_radius0=4, rs_steps=3),
                                dict(levels=1, n=3), dict(alpha=0.0), dict(seed=123456789012345),
                                dict(prop_scales=3), dict(p=3, prop_scales=4), dict(p=1, prop_scales=2)])
def test_nnf_estimate_config_variants(fb, ctx, kw):
    cfg, (sg, tg, ss, ts, keys), frames, tasks = _nnf_case(fb, 1, 40, 52, B=2, **kw)
    F, E, X, _ = ctx.fb_nnf_estimate(cfg, dev(sg), dev(tg), dev(ss), pair_keys=keys)
    Fr, Er, Xr, _ = O.nnf(ocfg(cfg), frames, tasks)
    assert_nnf(F, E, Fr, Er)
    assert_frames(X, Xr)


def test_nnf_batch_invariance(fb, ctx):
    cfg, (sg, tg, ss, ts, keys), frames, tasks = _nnf_case(fb, 1, 48, 48, B=4)
    Fb, Eb, Xb, _ = ctx.fb_nnf_estimate(cfg, dev(sg), dev(tg), dev(ss), pair_keys=keys)
    for b in (0, 3):
        F1, E1, X1, _ = ctx.fb_nnf_estimate(cfg, dev(sg[b:b + 1]), dev(tg[b:b + 1]), dev(ss[b:b + 1]),
                                            pair_keys=[keys[b]])
        assert torch.equal(F1[0], Fb[b]) and torch.equal(E1[0], Eb[b]) and torch.equal(X1[0], Xb[b])


def test_identical_frames_identity(fb, ctx):
    g = textured_frame(48, 40)[None].repeat(2, 0)
    cfg = fb.MatchCfg(patch_radius=2, iters_per_level=2, loss=fb.GUIDE_STYLE, init=fb.INIT_IDENTITY)
    F, E, X, _ = ctx.fb_nnf_estimate(cfg, dev(g), dev(g), dev(g), pair_keys=[(0, 1, 6), (0, 1, 6)])
    rr, cc = np.mgrid[0:48, 0:40]
    F = F.cpu().numpy()
    assert np.all(F[..., 0] == rr) and np.all(F[..., 1] == cc) and torch.all(E == 0)


# ------------------------------------------------------------------------------ a9/a10 window blends
CONFIG1 = dict(N=8, H=64, W=64, M=3, p=2, levels=2, n=2)  # BASELINE.json configs[0]


@pytest.mark.parametrize("mode", ["balanced", "accurate", "fast"])
def test_config1_blend_full_parity(fb, ctx, mode):
    c = CONFIG1
    g, s = moving_texture(c["N"], c["H"], c["W"])
    loss = fb.MEAN_ALIGN if mode == "accurate" else fb.GUIDE_STYLE
    sched = fb.TREE if mode == "fast" else fb.DIRECT
    cfg = fb.MatchCfg(patch_radius=c["p"], levels=c["levels"], iters_per_level=c["n"], loss=loss)
    out, st = ctx.fb_blend_window(cfg, sched, dev(g), dev(s), c["M"])
    fn = O.blend_tree if mode == "fast" else O.blend_direct
    ref, pairs, evals = fn(ocfg(cfg), g, s, c["M"])
    assert st["nnf_pairs"] == pairs == (28 if mode == "fast" else 36)
    assert st["candidate_evals"] == evals
    assert_frames(out, ref)


@pytest.mark.parametrize("N,M,H,W", [(1, 3, 32, 32), (5, 0, 32, 40), (6, 9, 24, 36), (11, 4, 37, 29)])
@pytest.mark.parametrize("mode", ["balanced", "accurate", "fast"])
def test_blend_edge_cases(fb, ctx, N, M, H, W, mode):
    g, s = moving_texture(N, H, W, seed=N * 7 + M)
    loss = fb.MEAN_ALIGN if mode == "accurate" else fb.GUIDE_STYLE
    sched = fb.TREE if mode == "fast" else fb.DIRECT
    cfg = fb.MatchCfg(patch_radius=2, iters_per_level=1, loss=loss)
    out, _ = ctx.fb_blend_window(cfg, sched, dev(g), dev(s), M)
    fn = O.blend_tree if mode == "fast" else O.blend_direct
    ref, _, _ = fn(ocfg(cfg), g, s, M)
    assert_frames(out, ref)
    if M == 0 or N == 1:
        assert_frames(out, s.astype(np.float32))


def test_constant_and_static_videos(fb, ctx):
    g, s = constant_video(6, 32, 40)
    for loss, sched in ((fb.GUIDE_STYLE, fb.DIRECT), (fb.MEAN_ALIGN, fb.DIRECT), (fb.GUIDE_STYLE, fb.TREE)):
        out, _ = ctx.fb_blend_window(fb.MatchCfg(iters_per_level=2, loss=loss), sched, dev(g), dev(s), 2)
        assert_frames(out, s.astype(np.float32))
    g, s = static_textured_video(9, 24, 28)
    cfg = fb.MatchCfg(iters_per_level=1, init=fb.INIT_IDENTITY)
    ref = np.stack([(s[max(0, i - 3):i + 4].astype(np.int64).sum(0) / (min(8, i + 3) - max(0, i - 3) + 1))
                    for i in range(9)]).astype(np.float32)
    for sched in (fb.DIRECT, fb.TREE):
        out, _ = ctx.fb_blend_window(cfg, sched, dev(g), dev(s), 3)
        assert_frames(out, ref)


@pytest.mark.parametrize("mode", ["balanced", "accurate", "fast"])
def test_batching_and_sharding_invariance(fb, mode):
    """Streaming (f4: batches of <= max_batch_pairs pairs, each with only its frames resident) and the
    shard entry point, every form against the oracle (not only against the single-batch GPU run)."""
    g, s = moving_texture(10, 40, 40, seed=31)
    loss = fb.MEAN_ALIGN if mode == "accurate" else fb.GUIDE_STYLE
    sched = fb.TREE if mode == "fast" else fb.DIRECT
    cfg = fb.MatchCfg(iters_per_level=1, loss=loss)
    M = 3
    ref, pairs, evals = (O.blend_tree if mode == "fast" else O.blend_direct)(ocfg(cfg), g, s, M)
    full, st = fb.Context(0).fb_blend_window(cfg, sched, dev(g), dev(s), M)
    assert st["nnf_pairs"] == pairs and st["candidate_evals"] == evals
    assert_frames(full, ref)
    for cap in (1, 5):
        small, st = fb.Context(0, max_batch_pairs=cap).fb_blend_window(cfg, sched, dev(g), dev(s), M)
        assert st["nnf_pairs"] == pairs
        assert_frames(small, ref)
    ctx = fb.Context(0, max_batch_pairs=4)
    for t0, t1 in ((0, 4), (4, 7), (7, 10)):
        f0, f1 = max(0, t0 - M), min(10, t1 + M)
        part, _ = ctx.fb_blend_window_range(cfg, sched, 10, f0, dev(g[f0:f1]), dev(s[f0:f1]), M, t0, t1)
        assert_frames(part, ref[t0:t1])


# ------------------------------------------------------------------------------ a11 interpolation
@pytest.mark.parametrize("keys", [[0, 7], [2, 5, 9], [4]])
def test_interpolation_parity(fb, ctx, keys):
    N = 10
    g, s = moving_texture(N, 40, 48, seed=17)
    cfg = fb.MatchCfg(iters_per_level=2)
    out, st = ctx.fb_interpolate_keyframes(cfg, dev(g), keys, dev(s[keys]))
    ref, pairs, evals = O.interpolate(ocfg(cfg), g, keys, s[keys])
    assert st["nnf_pairs"] == pairs and st["candidate_evals"] == evals
    assert_frames(out, ref)
    for k in keys:
        assert_frames(out[k], s[k].astype(np.float32))


# ------------------------------------------------------------------------------ errors
def test_error_statuses(fb, ctx):
    g, s = moving_texture(4, 32, 32)
    with pytest.raises(fb.FBError) as e:
        ctx.fb_blend_window(fb.MatchCfg(loss=fb.MEAN_ALIGN), fb.TREE, dev(g), dev(s), 2)
    assert e.value.status == 6
    with pytest.raises(fb.FBError) as e:
        ctx.fb_blend_window(fb.MatchCfg(patch_radius=9), fb.DIRECT, dev(g), dev(s), 2)
    assert e.value.status == 6
    with pytest.raises(fb.FBError) as e:
        ctx.fb_blend_window(fb.MatchCfg(patch_radius=3), fb.DIRECT, dev(g[:, :6, :6]), dev(s[:, :6, :6]), 2)
    assert e.value.status == 2
    with pytest.raises(fb.FBError) as e:
        ctx.fb_blend_window(fb.MatchCfg(), fb.DIRECT, dev(g), dev(s), -1)
    assert e.value.status == 1
    with pytest.raises(fb.FBError) as e:
        ctx.fb_interpolate_keyframes(fb.MatchCfg(), dev(g), [2, 1], dev(s[:2]))
    assert e.value.status == 1


def test_streaming_workspace_is_O_window(fb):
    """f4 / P:249: the direct schedule keeps only each batch's frames (+2M) resident, so the workspace of
    an accurate-mode blend does not grow with the video length once batches are capped."""
    ctx = fb.Context(0, max_batch_pairs=300)
    cfg = fb.MatchCfg(loss=fb.MEAN_ALIGN)
    w200 = ctx.workspace_size(fb.fb.OP_BLEND_DIRECT, cfg, 200, 512, 512, 15)
    w2000 = ctx.workspace_size(fb.fb.OP_BLEND_DIRECT, cfg, 2000, 512, 512, 15)
    assert w2000 == w200
    full = fb.Context(0).workspace_size(fb.fb.OP_BLEND_DIRECT, cfg, 2000, 512, 512, 15)
    assert w2000 < full / 5


# ------------------------------------------------------------------------------ f1 alignment (Eq. 10)
@pytest.mark.parametrize("p,H,W", [(2, 64, 64), (1, 45, 77), (2, 45, 77), (3, 40, 52)])
def test_pairwise_nnf_matches_oracle(fb, ctx, p, H, W):
    g, s = moving_texture(3, H, W, seed=21 + p)
    cfg = fb.MatchCfg(patch_radius=p, iters_per_level=2, loss=fb.PAIRWISE, alpha=4.0)
    sg = np.stack([g[0], g[2]])
    tg = np.stack([g[1], g[1]])
    ss = np.stack([s[0], s[2]])
    F, E, X, st = ctx.fb_nnf_estimate(cfg, dev(sg), dev(tg), dev(ss), group=[1, 0],
                                      pair_keys=[(0, 1, 5), (2, 1, 5)])
    frames = np.concatenate([g, s[[0, 2]]]).astype(np.float32)
    tasks = [dict(src_guide=0, tgt_guide=1, src_style=3, src_id=0, tgt_id=1, tag=5, partner=1),
             dict(src_guide=2, tgt_guide=1, src_style=4, src_id=2, tgt_id=1, tag=5, partner=0)]
    Fr, Er, Xr, ev = O.nnf(ocfg(cfg), frames, tasks)
    assert st["candidate_evals"] == ev
    assert_nnf(F, E, Fr, Er)
    assert_frames(X, Xr)


@pytest.mark.parametrize("keys", [[0, 7], [2, 5, 9], [4]])
def test_aligned_interpolation_parity(fb, ctx, keys):
    N = 10
    g, s = moving_texture(N, 40, 48, seed=18)
    cfg = fb.MatchCfg(iters_per_level=2, loss=fb.PAIRWISE)
    out, st = ctx.fb_interpolate_keyframes(cfg, dev(g), keys, dev(s[keys]))
    ref, pairs, evals = O.interpolate(ocfg(cfg), g, keys, s[keys])
    assert st["nnf_pairs"] == pairs and st["candidate_evals"] == evals
    assert_frames(out, ref)


def test_pairwise_rejects_bad_counterparts(fb, ctx):
    g, s = moving_texture(3, 32, 32)
    cfg = fb.MatchCfg(loss=fb.PAIRWISE)
    with pytest.raises(fb.FBError) as e:
        ctx.fb_nnf_estimate(cfg, dev(g[:2]), dev(g[1:]), dev(s[:2]), group=[1, 1], pair_keys=[(0, 1, 5), (2, 1, 5)])
    assert e.value.status == 1
    with pytest.raises(fb.FBError) as e:
        ctx.fb_blend_window(cfg, fb.DIRECT, dev(g), dev(s), 1)
    assert e.value.status == 1


@pytest.mark.parametrize("mode", ["balanced", "accurate", "fast"])
def test_jump_flood_blend_parity(fb, ctx, mode):
    """f3 / D41: jump-flood propagation (J = 3 scales) through every schedule."""
    g, s = moving_texture(7, 48, 40, seed=25)
    loss = fb.MEAN_ALIGN if mode == "accurate" else fb.GUIDE_STYLE
    sched = fb.TREE if mode == "fast" else fb.DIRECT
    cfg = fb.MatchCfg(iters_per_level=2, loss=loss, prop_scales=3)
    out, st = ctx.fb_blend_window(cfg, sched, dev(g), dev(s), 2)
    fn = O.blend_tree if mode == "fast" else O.blend_direct
    ref, pairs, evals = fn(ocfg(cfg), g, s, 2)
    assert st["candidate_evals"] == evals
    assert_frames(out, ref)


# ------------------------------------------------------------------------------ f2 tracking (D42)
@pytest.mark.parametrize("keys,align", [([0, 8], False), ([0, 8], True), ([3], False), ([1, 5, 9], True)])
def test_tracking_interpolation_parity(fb, ctx, keys, align):
    N = 10
    g, s = moving_texture(N, 40, 44, seed=27)
    cfg = fb.MatchCfg(iters_per_level=2, loss=fb.PAIRWISE if align else fb.GUIDE_STYLE, tracking=1)
    out, st = ctx.fb_interpolate_keyframes(cfg, dev(g), keys, dev(s[keys]))
    ref, pairs, evals = O.interpolate(ocfg(cfg), g, keys, s[keys])
    assert st["nnf_pairs"] == pairs and st["candidate_evals"] == evals
    assert_frames(out, ref)


# ------------------------------------------------------------------------------ schedule invariance / races
@pytest.mark.parametrize("mode", ["accurate", "fast"])
def test_fused_fields_equal_per_field_launches(fb, mode):
    """k_iter13_fast (fields 1-3 + random search in one launch, halo lanes) must equal the per-field launches
    (P:76 Jacobi fields) bit for bit, on every repetition: its halo lanes read the field-0 E of pixels owned
    by other tiles, so it must never write E in place (a timing-dependent race that this test repeats)."""
    g, s = moving_texture(6, 192, 160, seed=77)
    loss = fb.MEAN_ALIGN if mode == "accurate" else fb.GUIDE_STYLE
    sched = fb.TREE if mode == "fast" else fb.DIRECT
    cfg = fb.MatchCfg(iters_per_level=3, loss=loss)
    c0 = fb.Context(0)
    c0.set_option(fb.fb.OPT_FUSE13, 0)
    ref, _ = c0.fb_blend_window(cfg, sched, dev(g), dev(s), 3)
    c = fb.Context(0)
    for _ in range(4):
        out, _ = c.fb_blend_window(cfg, sched, dev(g), dev(s), 3)
        assert torch.equal(out, ref)



@pytest.mark.parametrize("N,M,world", [(12, 5, 3), (10, 3, 2), (9, 8, 3)])
def test_tree_cell_exchange_matches_full_blend(fb, N, M, world):
    """Sharded fast mode with blending-table cell exchange: every rank builds only the cells
    it owns, the cells move between ranks (here: within one process), and each rank's queries reproduce its
    targets of the single-call tree blend bit for bit."""
    from paper_2311_09265_b200 import shard
    g, s = moving_texture(N, 40, 48, seed=13)
    cfg = fb.MatchCfg(iters_per_level=1, loss=fb.GUIDE_STYLE)
    full, _ = fb.Context(0).fb_blend_window(cfg, fb.TREE, dev(g), dev(s), M)
    plan = shard.plan_shards(N, M, world, "tree")
    ctx = fb.Context(0)
    pool = {}
    for r in range(world):
        f0, f1 = shard.halo_range(N, M, *plan[r])
        build = shard.cells_to_build(plan, N, M, r)
        if build:
            T, _ = ctx.fb_tree_build_cells(cfg, N, f0, dev(g[f0:f1]), dev(s[f0:f1]), build)
            pool.update({c: T[k] for k, c in enumerate(build)})
    for r in range(world):
        t0, t1 = plan[r]
        f0, f1 = shard.halo_range(N, M, t0, t1)
        need = shard.tree_cells_needed(N, M, t0, t1)
        out, _ = ctx.fb_tree_query(cfg, N, f0, dev(g[f0:f1]), dev(s[f0:f1]), M, t0, t1, need, [pool[c] for c in need])
        assert torch.equal(out, full[t0:t1])
        ref, _, _ = O.blend_tree(ocfg(cfg), g, s, M, targets=list(range(t0, t1)))
        assert_frames(out, ref)
        if need:  # a query whose cells are incomplete is rejected, not silently wrong
            with pytest.raises(fb.FBError):
                ctx.fb_tree_query(cfg, N, f0, dev(g[f0:f1]), dev(s[f0:f1]), M, t0, t1, need[1:],
                                  [pool[c] for c in need[1:]])


@pytest.mark.parametrize("loss", ["GUIDE_STYLE", "PAIRWISE"])
def test_interpolation_range_equals_full_call(fb, loss):
    """Sharded interpolation: frames [t0, t1) from their own guides plus the broadcast keyframes
    equal the full call's rows bit for bit; tracking (D42) needs the full call."""
    from paper_2311_09265_b200 import shard
    N, keys = 11, [0, 5, 10]
    g, s = moving_texture(N, 36, 44, seed=21)
    ks = s[keys]
    cfg = fb.MatchCfg(iters_per_level=2, loss=getattr(fb, loss))
    ctx = fb.Context(0)
    full, _ = ctx.fb_interpolate_keyframes(cfg, dev(g), keys, dev(ks))
    ref, _, _ = O.interpolate(ocfg(cfg), g, keys, ks)
    assert_frames(full, ref)
    for t0, t1 in shard.plan_interp_shards(N, keys, 3) + [(2, 3), (5, 6)]:
        part, _ = ctx.fb_interpolate_keyframes_range(cfg, N, t0, t1, dev(g[t0:t1]), keys, dev(g[keys]), dev(ks))
        assert torch.equal(part, full[t0:t1])
        assert_frames(part, ref[t0:t1])
    cfg_t = fb.MatchCfg(iters_per_level=2, loss=fb.GUIDE_STYLE, tracking=1)
    with pytest.raises(fb.FBError):
        ctx.fb_interpolate_keyframes_range(cfg_t, N, 0, 4, dev(g[0:4]), keys, dev(g[keys]), dev(ks))


def test_context_on_a_side_stream(fb):
    """Results do not depend on the stream the context enqueues on (stream choice invariance)."""
    g, s = moving_texture(6, 48, 40, seed=8)
    cfg = fb.MatchCfg(iters_per_level=2, loss=fb.MEAN_ALIGN)
    ref, _ = fb.Context(0).fb_blend_window(cfg, fb.DIRECT, dev(g), dev(s), 2)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        c = fb.Context(0, stream=side)
        out, _ = c.fb_blend_window(cfg, fb.DIRECT, dev(g), dev(s), 2)
    side.synchronize()
    assert torch.equal(out, ref)


def test_context_stream_differs_from_current_stream(fb):
    """a context bound to a side stream, called while another stream is current: inputs copied and
    outputs allocated on the current stream must be ordered with the context's kernels (fb.py _ordered)."""
    g, s = moving_texture(6, 64, 48, seed=9)
    cfg = fb.MatchCfg(iters_per_level=2, loss=fb.MEAN_ALIGN)
    ref, _ = fb.Context(0).fb_blend_window(cfg, fb.DIRECT, dev(g), dev(s), 2)
    side = torch.cuda.Stream()
    c = fb.Context(0, stream=side)
    for _ in range(3):  # host tensors: the H2D copies run on the current stream, the kernels on `side`
        out, _ = c.fb_blend_window(cfg, fb.DIRECT, torch.from_numpy(g), torch.from_numpy(s), 2)
        assert torch.equal(out, ref)  # compared on the current stream without an explicit side.synchronize()


def test_mean_align_multi_group_fresh_context_workspace(fb):
    """fb_workspace_size(FB_OP_NNF) must cover one packed T-bar target per MEAN_ALIGN group."""
    g, s = moving_texture(5, 48, 40, seed=12)
    sg, tg = np.stack([g[0], g[2], g[1], g[3]]), np.stack([g[1], g[1], g[4], g[4]])
    ss, ts = np.stack([s[0], s[2], s[1], s[3]]), np.stack([s[1], s[1], s[4], s[4]])
    cfg = fb.MatchCfg(iters_per_level=2, loss=fb.MEAN_ALIGN)
    keys = [(0, 1, 0), (2, 1, 0), (1, 4, 0), (3, 4, 0)]
    F, E, X, st = fb.Context(0).fb_nnf_estimate(cfg, dev(sg), dev(tg), dev(ss), dev(ts), group=[0, 0, 1, 1],
                                                pair_keys=keys)
    frames = np.concatenate([g, s]).astype(np.float32)
    tasks = [dict(src_guide=a, tgt_guide=b, src_style=5 + a, tgt_style=5 + b, group=b, src_id=a, tgt_id=b, tag=0)
             for a, b, _ in keys]
    Fr, Er, Xr, ev = O.nnf(ocfg(cfg), frames, tasks)
    assert st["candidate_evals"] == ev
    assert_nnf(F, E, Fr, Er)
    assert_frames(X, Xr)


def test_invalid_iteration_and_step_counts_rejected(fb, ctx):
    """iters_per_level and rs_steps beyond the Philox counter fields (D21) are rejected."""
    g, s = moving_texture(3, 32, 32)
    for cfg in (fb.MatchCfg(iters_per_level=1024), fb.MatchCfg(rs_steps=4096)):
        with pytest.raises(fb.FBError) as e:
            ctx.fb_blend_window(cfg, fb.DIRECT, dev(g), dev(s), 1)
        assert e.value.status == 1


@pytest.mark.parametrize("mode,H,W", [("accurate", 96, 80), ("balanced", 128, 112), ("accurate", 135, 67)])
def test_level1_fast_path_matches_oracle(fb, mode, H, W):
    """Level 1 of u8 sources runs through the 16-byte TF10 target and the fused kernels (FB_OPT_L1_FAST): the
    FP32 chains on exact biased operands must equal the oracle bit for bit, and equal the general kernel."""
    g, s = moving_texture(5, H, W, seed=41)
    loss = fb.MEAN_ALIGN if mode == "accurate" else fb.GUIDE_STYLE
    cfg = fb.MatchCfg(iters_per_level=2, loss=loss, levels=3 if H == 135 else 0)
    ctx = fb.Context(0)
    ctx.set_option(fb.fb.OPT_L1_FAST, 1)
    out, st = ctx.fb_blend_window(cfg, fb.DIRECT, dev(g), dev(s), 2)
    ref, pairs, evals = O.blend_direct(ocfg(cfg), g, s, 2)
    assert st["candidate_evals"] == evals
    assert_frames(out, ref)
    c2 = fb.Context(0)
    c2.set_option(fb.fb.OPT_L1_FAST, 0)
    out2, _ = c2.fb_blend_window(cfg, fb.DIRECT, dev(g), dev(s), 2)
    assert torch.equal(out, out2)


@pytest.mark.parametrize("l1_fast", [0, 1])
def test_level1_fast_path_nnf_and_error(fb, l1_fast):
    """NNF and E after a 3-level estimation (levels 2 -> 1 -> 0) through fb_nnf_estimate, against the oracle."""
    ctx = fb.Context(0)
    ctx.set_option(fb.fb.OPT_L1_FAST, l1_fast)
    g, s = moving_texture(3, 72, 88, seed=43)
    cfg = fb.MatchCfg(iters_per_level=2, loss=fb.GUIDE_STYLE, levels=3)
    F, E, X, st = ctx.fb_nnf_estimate(cfg, dev(g[[0, 2]]), dev(g[[1, 1]]), dev(s[[0, 2]]), pair_keys=[(0, 1, 0), (2, 1, 0)])
    frames = np.concatenate([g, s]).astype(np.float32)
    tasks = [dict(src_guide=0, tgt_guide=1, src_style=3, src_id=0, tgt_id=1, tag=0),
             dict(src_guide=2, tgt_guide=1, src_style=5, src_id=2, tgt_id=1, tag=0)]
    Fr, Er, Xr, ev = O.nnf(ocfg(cfg), frames, tasks)
    assert st["candidate_evals"] == ev
    assert_nnf(F, E, Fr, Er)
    assert_frames(X, Xr)


@pytest.mark.parametrize("loss,H,W,sb,l1,rows", [(1, 96, 112, 1, 0, 1), (2, 96, 112, 1, 0, 1), (0, 64, 80, 1, 0, 1),
                                                 (1, 96, 112, 0, 0, 1), (2, 135, 67, 1, 1, 1), (1, 128, 112, 1, 1, 1),
                                                 (2, 96, 112, 1, 0, 0), (2, 96, 112, 1, 0, 2), (1, 67, 135, 1, 0, 2),
                                                 (2, 96, 112, 1, 0, 3), (0, 64, 80, 1, 0, 3)])
def test_patch_sum_bound_matches_oracle(fb, loss, H, W, sb, l1, rows):
    """The random search's patch-sum bound (FB_OPT_SUM_BOUND) only skips candidates that provably
    lose the strict select: NNF and E equal the oracle bit for bit with the bound on and off, at level 0 and, with
    FB_OPT_L1_FAST, at level 1, for every count of target rows held in registers; odd sizes put candidates on the
    zero-padded border."""
    c = fb.Context(0)
    c.set_option(fb.fb.OPT_SUM_BOUND, sb)
    c.set_option(fb.fb.OPT_L1_FAST, l1)
    c.set_option(fb.fb.OPT_TGT_REG_ROWS, rows)
    cfg, (sg, tg, ss, ts, keys), frames, tasks = _nnf_case(fb, loss, H, W, seed=47, n=3, levels=3)
    group = [0] * len(keys) if loss == fb.MEAN_ALIGN else None
    F, E, X, st = c.fb_nnf_estimate(cfg, dev(sg), dev(tg), None if loss == 0 else dev(ss),
                                    dev(ts) if loss == 2 else None, group=group, pair_keys=keys)
    Fr, Er, Xr, ev = O.nnf(ocfg(cfg), frames, tasks, want_x=loss != 0)
    assert st["candidate_evals"] == ev
    assert_nnf(F, E, Fr, Er)
    if loss != 0:
        assert_frames(X, Xr)


@pytest.mark.parametrize("loss,H,W,tail", [(2, 96, 112, 1), (1, 135, 67, 1), (2, 67, 135, 0), (1, 96, 112, 0),
                                            (2, 160, 192, 1)])
def test_tail_bound_matches_oracle(fb, loss, H, W, tail):
    """The fused level-0 random search's partial + remainder bound (FB_OPT_TAIL_BOUND: FP32 partial
    of the first three patch rows plus Cauchy-Schwarz on the last two rows' sums) only skips candidates that
    provably lose: NNF, E and the candidate count equal the oracle's bit for bit with the bound on and off, odd
    sizes putting tail rows on the zero-padded border."""
    c = fb.Context(0)
    c.set_option(fb.fb.OPT_TAIL_BOUND, tail)
    cfg, (sg, tg, ss, ts, keys), frames, tasks = _nnf_case(fb, loss, H, W, seed=61, n=3, levels=3)
    group = [0] * len(keys) if loss == fb.MEAN_ALIGN else None
    F, E, X, st = c.fb_nnf_estimate(cfg, dev(sg), dev(tg), dev(ss), dev(ts) if loss == 2 else None, group=group,
                                    pair_keys=keys)
    Fr, Er, Xr, ev = O.nnf(ocfg(cfg), frames, tasks, want_x=True)
    assert st["candidate_evals"] == ev
    assert_nnf(F, E, Fr, Er)
    assert_frames(X, Xr)


@pytest.mark.parametrize("sb,rows", [(0, 1), (1, 1), (1, 3)])
def test_patch_sum_bound_tree_blend(fb, sb, rows):
    """Fast mode: the tree queries' float-style sources (SF8F blending-table cells) carry FP32 patch sums with an
    absolute margin; the blend equals the oracle bit for bit with the bound on and off."""
    c = fb.Context(0)
    c.set_option(fb.fb.OPT_SUM_BOUND, sb)
    c.set_option(fb.fb.OPT_TGT_REG_ROWS, rows)
    g, s = moving_texture(9, 72, 96, seed=53)
    cfg = fb.MatchCfg(iters_per_level=3, loss=fb.GUIDE_STYLE, levels=2)
    out, st = c.fb_blend_window(cfg, fb.TREE, dev(g), dev(s), 4)
    ref, pairs, evals = O.blend_tree(ocfg(cfg), g, s, 4)
    assert st["candidate_evals"] == evals
    assert_frames(out, ref)


@pytest.mark.parametrize("mode", ["balanced", "accurate"])
def test_blend_tracking_parity(fb, ctx, mode):
    """Tracking in blending (P:259 optional setting, D44): every pair NNF(G_j, G_i) also tries NNF(G_j, G_{i+-1});
    the direct blend equals the oracle bit for bit and evaluates exactly the oracle's candidate count."""
    g, s = moving_texture(7, 40, 48, seed=57)
    cfg = fb.MatchCfg(iters_per_level=2, loss=fb.MEAN_ALIGN if mode == "accurate" else fb.GUIDE_STYLE, tracking=1)
    out, st = ctx.fb_blend_window(cfg, fb.DIRECT, dev(g), dev(s), 2)
    ref, pairs, evals = O.blend_direct(ocfg(cfg), g, s, 2)
    assert st["nnf_pairs"] == pairs and st["candidate_evals"] == evals
    assert_frames(out, ref)


def test_blend_tracking_unsupported_forms(fb, ctx):
    """D44 couples every pair of the schedule: the tree schedule and partial ranges are rejected."""
    g, s = moving_texture(6, 32, 32, seed=58)
    cfg = fb.MatchCfg(iters_per_level=1, tracking=1)
    with pytest.raises(fb.FBError) as e:
        ctx.fb_blend_window(cfg, fb.TREE, dev(g), dev(s), 2)
    assert e.value.status == 6
    with pytest.raises(fb.FBError) as e:
        ctx.fb_blend_window_range(cfg, fb.DIRECT, 6, 0, dev(g), dev(s), 2, 0, 3)
    assert e.value.status == 6


@pytest.mark.parametrize("mode", ["accurate", "fast"])
def test_max_size_identical_frames_identity(fb, mode):
    """Largest frames in the tests (UHD 2160x3840, 7 pyramid levels): with identity init on identical frames every
    NNF stays the identity (E = 0 is never beaten, D16), so the blend returns the style exactly (P6 at full scale;
    exercises the 64-bit offsets, slot pitches and patch-sum planes at the largest sizes)."""
    g1 = textured_frame(2160, 3840, seed=61)
    g = np.stack([g1, g1, g1])
    s = np.stack([g1[..., ::-1], g1[..., ::-1], g1[..., ::-1]]).copy()
    loss = fb.MEAN_ALIGN if mode == "accurate" else fb.GUIDE_STYLE
    cfg = fb.MatchCfg(iters_per_level=1, loss=loss, init=fb.INIT_IDENTITY)
    out, st = fb.Context(0).fb_blend_window(cfg, fb.TREE if mode == "fast" else fb.DIRECT, dev(g), dev(s), 1)
    assert st["nnf_pairs"] > 0
    assert torch.equal(out, dev(s).float())


@pytest.mark.parametrize("mode,p3f", [("balanced", 1), ("accurate", 1), ("balanced", 0)])
def test_p3_fused_fields_match_oracle(fb, mode, p3f):
    """p = 3 (config 5's patch 7) at level 0: fields 1-3 and the random search in one launch (FB_OPT_P3_FUSED) or as
    separate launches, both equal to the oracle bit for bit on a ragged size."""
    c = fb.Context(0)
    c.set_option(fb.fb.OPT_P3_FUSED, p3f)
    g, s = moving_texture(5, 70, 101, seed=63)
    cfg = fb.MatchCfg(patch_radius=3, iters_per_level=2, loss=fb.MEAN_ALIGN if mode == "accurate" else fb.GUIDE_STYLE)
    out, st = c.fb_blend_window(cfg, fb.DIRECT, dev(g), dev(s), 2)
    ref, pairs, evals = O.blend_direct(ocfg(cfg), g, s, 2)
    assert st["candidate_evals"] == evals
    assert_frames(out, ref)


@pytest.mark.parametrize("H,W,loss", [(5, 5, 2), (5, 203, 1), (203, 5, 2), (6, 33, 1), (31, 7, 0)])
def test_extreme_shapes_match_oracle(fb, ctx, H, W, loss):
    """Smallest and most elongated frames for p = 2 (one pyramid level, a single ragged tile in one dimension):
    NNF, E and remap equal the oracle bit for bit."""
    cfg, (sg, tg, ss, ts, keys), frames, tasks = _nnf_case(fb, loss, H, W, seed=67, n=3)
    group = [0] * len(keys) if loss == fb.MEAN_ALIGN else None
    F, E, X, st = ctx.fb_nnf_estimate(cfg, dev(sg), dev(tg), None if loss == 0 else dev(ss),
                                      dev(ts) if loss == 2 else None, group=group, pair_keys=keys)
    Fr, Er, Xr, ev = O.nnf(ocfg(cfg), frames, tasks, want_x=loss != 0)
    assert st["candidate_evals"] == ev
    assert_nnf(F, E, Fr, Er)
    if loss != 0:
        assert_frames(X, Xr)
