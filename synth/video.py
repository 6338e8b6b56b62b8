"""Seeded synthetic videos.

``moving_texture(N, H, W)`` returns (guide, style) uint8 [N,H,W,3]:

* canvas: fBm value noise, 5 octaves at cell sizes 64..4 px, amplitude halving per octave,
  independent RGB fields, plus 24 flat-colour rectangles / discs for hard edges, normalised to 0..255;
  the canvas exceeds the frame by the total camera motion;
* guide frame t: a crop at (round(v_r t), round(v_c t)), v ~ U[-1.5, 1.5] px/frame, with 4 textured disc
  sprites (radius 5-12 % of H) moving at U[-3, 3] px/frame (occlusions) and a global gain
  1 + 0.02 sin(2 pi t / 50); quantised with round-half-even;
* style frame t: a fixed stylisation of G_t (per-channel gamma and contrast, channel rotation) plus
  flicker: a bilinear-upsampled 8x8x3 field U[-25, 25] seeded by (seed, t) and i.i.d. U[-4, 4]; clipped
  and quantised.  This is the "diffusion-rendered frames flicker" situation of P:106-113.
"""
from __future__ import annotations

import numpy as np

SEED_VIDEO = 20231116


def _bilinear(grid: np.ndarray, h: int, w: int, cell: float) -> np.ndarray:
    """Upsample grid [gh, gw, C] to [h, w, C]; sample (r, c) sits at (r/cell, c/cell) in grid units."""
    gh, gw = grid.shape[:2]
    ry = np.arange(h, dtype=np.float64) / cell
    rx = np.arange(w, dtype=np.float64) / cell
    y0 = np.minimum(np.floor(ry).astype(np.int64), gh - 2)
    x0 = np.minimum(np.floor(rx).astype(np.int64), gw - 2)
    fy = (ry - y0)[:, None, None]
    fx = (rx - x0)[None, :, None]
    fy = fy * fy * (3 - 2 * fy)  # smoothstep: value noise without grid creases
    fx = fx * fx * (3 - 2 * fx)
    g00 = grid[y0][:, x0]
    g01 = grid[y0][:, x0 + 1]
    g10 = grid[y0 + 1][:, x0]
    g11 = grid[y0 + 1][:, x0 + 1]
    return (g00 * (1 - fy) * (1 - fx) + g01 * (1 - fy) * fx + g10 * fy * (1 - fx) + g11 * fy * fx)


def _fbm(rng: np.random.Generator, h: int, w: int, cells=(64, 32, 16, 8, 4)) -> np.ndarray:
    out = np.zeros((h, w, 3), np.float64)
    amp = 1.0
    for cell in cells:
        grid = rng.random((h // cell + 3, w // cell + 3, 3))
        out += amp * _bilinear(grid, h, w, float(cell))
        amp *= 0.5
    return out


def _shapes(rng: np.random.Generator, img: np.ndarray, count: int = 24) -> None:
    h, w, _ = img.shape
    yy, xx = np.mgrid[0:h, 0:w]
    lo, hi = img.min(), img.max()
    for _ in range(count):
        col = lo + (hi - lo) * rng.random(3)
        cy, cx = rng.integers(0, h), rng.integers(0, w)
        size = rng.integers(max(2, min(h, w) // 40), max(3, min(h, w) // 8))
        if rng.random() < 0.5:
            m = (np.abs(yy - cy) <= size) & (np.abs(xx - cx) <= size * (0.5 + rng.random()))
        else:
            m = (yy - cy) ** 2 + (xx - cx) ** 2 <= size * size
        img[m] = col


def _normalise(img: np.ndarray) -> np.ndarray:
    lo, hi = img.min(), img.max()
    return (img - lo) * (255.0 / max(hi - lo, 1e-9))


def _quant(x: np.ndarray) -> np.ndarray:
    return np.clip(np.rint(x), 0, 255).astype(np.uint8)  # np.rint = round-half-even


def moving_texture(N: int, H: int, W: int, seed: int = SEED_VIDEO, n_sprites: int = 4, t0: int = 0,
                   t1: int | None = None):
    """(guide, style) uint8 [N, H, W, 3] — the synthetic workload of DESIGN.md §5.  With t0/t1 only frames
    [t0, t1) of the N-frame video are generated (identical to the same rows of the full call: a frame depends
    only on its index and the video-wide draws), so a shard can build just its own frames."""
    t1 = N if t1 is None else t1
    rng = np.random.default_rng(seed)
    v = rng.uniform(-1.5, 1.5, size=2)
    span = np.abs(v) * max(N - 1, 0)
    pad_r, pad_c = int(np.ceil(span[0])) + 2, int(np.ceil(span[1])) + 2
    ch, cw = H + 2 * pad_r, W + 2 * pad_c
    canvas = _fbm(rng, ch, cw)
    _shapes(rng, canvas)
    canvas = _normalise(canvas)
    # sprites: textured discs with their own noise texture
    sprites = []
    for _ in range(n_sprites):
        rad = int(max(2, round(H * rng.uniform(0.05, 0.12))))
        tex = _normalise(_fbm(rng, 2 * rad + 1, 2 * rad + 1, cells=(8, 4, 2)) + rng.random(3) * 2)
        yy, xx = np.mgrid[-rad:rad + 1, -rad:rad + 1]
        mask = yy * yy + xx * xx <= rad * rad
        p0 = rng.uniform([0, 0], [H, W])
        vel = rng.uniform(-3, 3, size=2)
        sprites.append((rad, tex, mask, p0, vel))
    # stylisation parameters (fixed for the whole video)
    gamma = rng.uniform(0.6, 1.6, size=3)
    contrast = rng.uniform(0.8, 1.3, size=3)
    rot = int(rng.integers(1, 3))
    guide = np.empty((t1 - t0, H, W, 3), np.uint8)
    style = np.empty((t1 - t0, H, W, 3), np.uint8)
    for t in range(t0, t1):
        o_r = pad_r + int(np.rint(v[0] * t))
        o_c = pad_c + int(np.rint(v[1] * t))
        frame = canvas[o_r:o_r + H, o_c:o_c + W].copy()
        for rad, tex, mask, p0, vel in sprites:
            cy = int(np.rint(p0[0] + vel[0] * t)) % (H + 2 * rad) - rad
            cx = int(np.rint(p0[1] + vel[1] * t)) % (W + 2 * rad) - rad
            y0, y1 = max(cy - rad, 0), min(cy + rad + 1, H)
            x0, x1 = max(cx - rad, 0), min(cx + rad + 1, W)
            if y0 >= y1 or x0 >= x1:
                continue
            sub_m = mask[y0 - (cy - rad):y1 - (cy - rad), x0 - (cx - rad):x1 - (cx - rad)]
            sub_t = tex[y0 - (cy - rad):y1 - (cy - rad), x0 - (cx - rad):x1 - (cx - rad)]
            frame[y0:y1, x0:x1][sub_m] = sub_t[sub_m]
        frame = frame * (1.0 + 0.02 * np.sin(2 * np.pi * t / 50.0))
        g = _quant(frame)
        guide[t - t0] = g
        x = g.astype(np.float64) / 255.0
        s = 255.0 * np.clip((x ** gamma - 0.5) * contrast + 0.5, 0, 1)
        s = np.roll(s, rot, axis=2)
        frng = np.random.default_rng([seed, t])
        field = _bilinear(frng.uniform(-25, 25, size=(8 + 1, 8 + 1, 3)), H, W, H / 8.0)
        s = s + field + frng.uniform(-4, 4, size=s.shape)
        style[t - t0] = _quant(s)
    return guide, style


# ---------------------------------------------------------------- pin fixtures

def constant_video(N: int, H: int, W: int, value=(90, 160, 30)):
    g = np.empty((N, H, W, 3), np.uint8)
    g[...] = np.asarray(value, np.uint8)
    s = np.empty_like(g)
    s[...] = np.asarray(value[::-1], np.uint8)
    return g, s


def static_textured_video(N: int, H: int, W: int, seed: int = 7, flicker: bool = True):
    """One textured guide frame repeated N times; style = per-frame random texture (if flicker)."""
    rng = np.random.default_rng(seed)
    g0 = _quant(_normalise(_fbm(rng, H, W, cells=(8, 4, 2)) + rng.random((H, W, 3))))
    guide = np.broadcast_to(g0, (N, H, W, 3)).copy()
    if flicker:
        style = rng.integers(0, 256, size=(N, H, W, 3), dtype=np.uint8)
    else:
        style = guide.copy()
    return guide, style


def iid_frames(n: int, H: int, W: int, seed: int = 3):
    rng = np.random.default_rng(seed)
    return rng.integers(0, 256, size=(n, H, W, 3), dtype=np.uint8)


def textured_frame(H: int, W: int, seed: int = 11) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return _quant(_normalise(_fbm(rng, H, W, cells=(16, 8, 4, 2)) + 0.5 * rng.random((H, W, 3))))
