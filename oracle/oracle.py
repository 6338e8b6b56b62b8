"""ctypes marshalling for the C oracle (fb_oracle.c).  TEST INFRASTRUCTURE ONLY (see __init__)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fb_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
# ORACLE_LIB: load a prebuilt oracle library instead (tools/oracle_mutations.py runs the pins against
# deliberately broken builds to show that each pin catches its mistake)
_LIB_OVERRIDE = os.environ.get("ORACLE_LIB")

# -O2, no fast-math, no FP contraction: the only fused ops are the explicit fmaf() calls (D20).
CFLAGS = ["-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off", "-fno-fast-math"]

BASE, GUIDE_STYLE, MEAN_ALIGN, PAIRWISE = 0, 1, 2, 3
INIT_RANDOM, INIT_IDENTITY = 0, 1
TAG_DIRECT, TAG_TREE_BUILD_F, TAG_TREE_QUERY_F, TAG_TREE_BUILD_R, TAG_TREE_QUERY_R, TAG_INTERP, TAG_API = range(7)


def build(force: bool = False) -> str:
    """Compile the oracle (gcc).  Called by __graft_entry__.build() and lazily by load()."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Cfg(C.Structure):
    _fields_ = [("patch_radius", C.c_int32), ("levels", C.c_int32), ("iters_per_level", C.c_int32),
                ("rs_radius0", C.c_int32), ("rs_steps", C.c_int32), ("alpha", C.c_float),
                ("loss", C.c_int32), ("init", C.c_int32), ("seed", C.c_uint64), ("prop_scales", C.c_int32),
                ("tracking", C.c_int32)]


class _Task(C.Structure):
    _fields_ = [("src_guide", C.c_int), ("tgt_guide", C.c_int), ("src_style", C.c_int), ("tgt_style", C.c_int),
                ("group", C.c_int), ("src_id", C.c_int), ("tgt_id", C.c_int), ("tag", C.c_int),
                ("partner", C.c_int), ("track_prev", C.c_int), ("track_next", C.c_int)]


@dataclass
class Cfg:
    """PatchMatch configuration (D1, D6, D13-D15, D21, D33)."""
    patch_radius: int = 2
    levels: int = 0
    iters_per_level: int = 5
    rs_radius0: int = 0
    rs_steps: int = 0
    alpha: float = 10.0
    loss: int = GUIDE_STYLE
    init: int = INIT_RANDOM
    seed: int = 1
    prop_scales: int = 1
    tracking: int = 0

    def c(self) -> _Cfg:
        return _Cfg(self.patch_radius, self.levels, self.iters_per_level, self.rs_radius0, self.rs_steps,
                    self.alpha, self.loss, self.init, self.seed, self.prop_scales, self.tracking)


_lib = None


def load():
    global _lib
    if _lib is None:
        _lib = C.CDLL(_LIB_OVERRIDE or build())
        P = C.POINTER
        _lib.orc_philox4x32_10.argtypes = [P(C.c_uint32), P(C.c_uint32), P(C.c_uint32)]
        _lib.orc_level_count.argtypes = [C.c_int] * 4
        _lib.orc_pyramid_pixels.restype = C.c_size_t
        _lib.orc_pyramid_pixels.argtypes = [C.c_int] * 3
        _lib.orc_pyramid.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
        _lib.orc_patch_dist.restype = C.c_float
        _lib.orc_patch_dist.argtypes = [C.c_void_p, C.c_void_p] + [C.c_int] * 7
        _lib.orc_remap.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p]
        _lib.orc_evals_per_task.restype = C.c_uint64
        _lib.orc_evals_per_task.argtypes = [P(_Cfg), C.c_int, C.c_int]
        _lib.orc_nnf.argtypes = [P(_Cfg), C.c_int, C.c_int, C.c_int, C.c_void_p, P(_Task), C.c_void_p, C.c_void_p,
                                 C.c_void_p, P(C.c_uint64)]
        _lib.orc_blend_direct.argtypes = [P(_Cfg), C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                          C.c_int, C.c_void_p, C.c_void_p, P(C.c_uint64), P(C.c_uint64)]
        _lib.orc_blend_tree.argtypes = _lib.orc_blend_direct.argtypes
        _lib.orc_interpolate.argtypes = [P(_Cfg), C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p,
                                         C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, P(C.c_uint64), P(C.c_uint64)]
        _lib.orc_tree_query_nodes.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        _lib.orc_tree_build_tasks.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.orc_field.argtypes = [P(_Cfg), C.c_int, C.c_int] + [C.c_void_p] * 4 + [C.c_int] * 6 + [C.c_void_p] * 2
        _lib.orc_set_threads.argtypes = [C.c_int]
        _lib.orc_track_field.argtypes = [P(_Cfg), C.c_int, C.c_int] + [C.c_void_p] * 7
        _lib.orc_upsample.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int]
        _lib.orc_field_step.argtypes = [P(_Cfg), C.c_int, C.c_int] + [C.c_void_p] * 4 + [C.c_int] * 7 + [C.c_void_p] * 2
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def num_threads() -> int:
    return int(load().orc_num_threads())


def set_threads(n: int) -> None:
    load().orc_set_threads(int(n))


def philox4x32_10(ctr, key):
    ctr_a = (C.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in ctr])
    key_a = (C.c_uint32 * 2)(*[int(x) & 0xFFFFFFFF for x in key])
    out = (C.c_uint32 * 4)()
    load().orc_philox4x32_10(ctr_a, key_a, out)
    return [int(x) for x in out]


def level_count(H: int, W: int, p: int, requested: int = 0) -> int:
    return int(load().orc_level_count(H, W, p, requested))


def pyramid(img: np.ndarray, levels: int) -> list[np.ndarray]:
    """img float32 [H,W,3] -> [level0, level1, ...] (D6)."""
    img = np.ascontiguousarray(img, dtype=np.float32)
    H, W, _ = img.shape
    out = np.zeros(3 * load().orc_pyramid_pixels(H, W, levels), np.float32)
    load().orc_pyramid(_p(img), H, W, levels, _p(out))
    res, off = [], 0
    for k in range(levels):
        n = (H >> k) * (W >> k) * 3
        res.append(out[off:off + n].reshape(H >> k, W >> k, 3))
        off += n
    return res


def patch_dist(A: np.ndarray, B: np.ndarray, sr: int, sc: int, r: int, c: int, p: int) -> np.float32:
    A = np.ascontiguousarray(A, np.float32)
    B = np.ascontiguousarray(B, np.float32)
    assert A.shape == B.shape
    h, w, _ = A.shape
    return np.float32(load().orc_patch_dist(_p(A), _p(B), h, w, sr, sc, r, c, p))


def remap(S: np.ndarray, F: np.ndarray, p: int) -> np.ndarray:
    S = np.ascontiguousarray(S, np.float32)
    F = np.ascontiguousarray(F, np.int32)
    h, w, _ = S.shape
    out = np.zeros_like(S)
    load().orc_remap(_p(S), h, w, _p(F), p, _p(out))
    return out


def upsample(Fc: np.ndarray, h: int, w: int) -> np.ndarray:
    """Alg. 1 "Upsample F" (D7): coarse NNF int32 [hc,wc,2] -> fine NNF int32 [h,w,2]."""
    Fc = np.ascontiguousarray(Fc, np.int32)
    hc, wc, _ = Fc.shape
    Ff = np.zeros((h, w, 2), np.int32)
    load().orc_upsample(_p(Fc), hc, wc, _p(Ff), h, w)
    return Ff


def evals_per_task(cfg: Cfg, H: int, W: int) -> int:
    cc = cfg.c()
    return int(load().orc_evals_per_task(C.byref(cc), H, W))


def nnf(cfg: Cfg, frames: np.ndarray, tasks: list[dict], want_x: bool = True):
    """frames float32 [NF,H,W,3]; tasks: dicts with src_guide, tgt_guide, src_style, tgt_style, group,
    src_id, tgt_id, tag, partner (PAIRWISE counterpart task index).  Returns (F [T,H,W,2] int32, E [T,H,W] float32, X [T,H,W,3] or None, evals)."""
    frames = np.ascontiguousarray(frames, np.float32)
    _, H, W, _ = frames.shape
    T = len(tasks)
    arr = (_Task * max(T, 1))()
    for i, t in enumerate(tasks):
        arr[i] = _Task(t["src_guide"], t["tgt_guide"], t.get("src_style", -1), t.get("tgt_style", -1),
                       t.get("group", i), t.get("src_id", 0), t.get("tgt_id", 0), t.get("tag", TAG_API),
                       t.get("partner", -1), t.get("track_prev", -1), t.get("track_next", -1))
    F = np.zeros((T, H, W, 2), np.int32)
    E = np.zeros((T, H, W), np.float32)
    X = np.zeros((T, H, W, 3), np.float32) if want_x else None
    ev = C.c_uint64(0)
    cc = cfg.c()
    rc = load().orc_nnf(C.byref(cc), T, H, W, _p(frames), arr, _p(F), _p(E), _p(X) if want_x else None,
                        C.byref(ev))
    if rc != 0:
        raise ValueError("orc_nnf: invalid shape for patch radius / levels")
    return F, E, X, int(ev.value)


def _targets(N, targets):
    t = np.arange(N, dtype=np.int32) if targets is None else np.ascontiguousarray(targets, np.int32)
    return t


def blend_direct(cfg: Cfg, guide: np.ndarray, style: np.ndarray, M: int, targets=None):
    """Balanced (cfg.loss=GUIDE_STYLE) or accurate (cfg.loss=MEAN_ALIGN) window blend, O(N*M)."""
    guide = np.ascontiguousarray(guide, np.uint8)
    style = np.ascontiguousarray(style, np.uint8)
    N, H, W, _ = guide.shape
    t = _targets(N, targets)
    out = np.zeros((len(t), H, W, 3), np.float32)
    pairs, evals = C.c_uint64(0), C.c_uint64(0)
    cc = cfg.c()
    rc = load().orc_blend_direct(C.byref(cc), N, H, W, M, _p(guide), _p(style), len(t), _p(t), _p(out),
                                 C.byref(pairs), C.byref(evals))
    if rc != 0:
        raise ValueError("orc_blend_direct failed")
    return out, int(pairs.value), int(evals.value)


def blend_tree(cfg: Cfg, guide: np.ndarray, style: np.ndarray, M: int, targets=None):
    """Fast mode: Alg. 3-5 + Eq. 6 (GUIDE_STYLE loss, D22)."""
    guide = np.ascontiguousarray(guide, np.uint8)
    style = np.ascontiguousarray(style, np.uint8)
    N, H, W, _ = guide.shape
    t = _targets(N, targets)
    out = np.zeros((len(t), H, W, 3), np.float32)
    pairs, evals = C.c_uint64(0), C.c_uint64(0)
    cc = cfg.c()
    rc = load().orc_blend_tree(C.byref(cc), N, H, W, M, _p(guide), _p(style), len(t), _p(t), _p(out),
                               C.byref(pairs), C.byref(evals))
    if rc != 0:
        raise ValueError("orc_blend_tree failed")
    return out, int(pairs.value), int(evals.value)


def interpolate(cfg: Cfg, guide: np.ndarray, key_index, key_style: np.ndarray, targets=None):
    guide = np.ascontiguousarray(guide, np.uint8)
    key_style = np.ascontiguousarray(key_style, np.uint8)
    N, H, W, _ = guide.shape
    ki = np.ascontiguousarray(key_index, np.int32)
    t = _targets(N, targets)
    out = np.zeros((len(t), H, W, 3), np.float32)
    pairs, evals = C.c_uint64(0), C.c_uint64(0)
    cc = cfg.c()
    rc = load().orc_interpolate(C.byref(cc), N, H, W, _p(guide), len(ki), _p(ki), _p(key_style), len(t), _p(t),
                                _p(out), C.byref(pairs), C.byref(evals))
    if rc != 0:
        raise ValueError("orc_interpolate failed")
    return out, int(pairs.value), int(evals.value)


def tree_query_nodes(l: int, r: int):
    n = np.zeros(64, np.int32)
    lv = np.zeros(64, np.int32)
    k = load().orc_tree_query_nodes(l, r, _p(n), _p(lv))
    return list(zip(n[:k].tolist(), lv[:k].tolist()))


def tree_build_tasks(N: int, lcap: int):
    k = load().orc_tree_build_tasks(N, lcap, None, None, None)
    s = np.zeros(max(k, 1), np.int32)
    d = np.zeros(max(k, 1), np.int32)
    lv = np.zeros(max(k, 1), np.int32)
    load().orc_tree_build_tasks(N, lcap, _p(s), _p(d), _p(lv))
    return list(zip(s[:k].tolist(), d[:k].tolist(), lv[:k].tolist()))


def field(cfg: Cfg, sg, tg, F, E, field_id: int, ss=None, aux=None, k: int = 0, it: int = 0,
          src_id: int = 0, tgt_id: int = 0, tag: int = TAG_API, step: int = 1):
    """One element of Alg. 1's updating sequence at a single level (field -1 = E init, 0..3 =
    propagation directions, 4+s = random-search step s).  Returns the updated (F, E)."""
    sg = np.ascontiguousarray(sg, np.float32)
    tg = np.ascontiguousarray(tg, np.float32)
    h, w, _ = sg.shape
    F = np.array(F, np.int32, copy=True, order="C")
    E = np.array(E, np.float32, copy=True, order="C")
    ss_ = None if ss is None else np.ascontiguousarray(ss, np.float32)
    aux_ = None if aux is None else np.ascontiguousarray(aux, np.float32)
    cc = cfg.c()
    load().orc_field_step(C.byref(cc), h, w, _p(sg), _p(tg), None if ss_ is None else _p(ss_),
                          None if aux_ is None else _p(aux_), field_id, step, k, it, src_id, tgt_id, tag, _p(F), _p(E))
    return F, E


def track_field(cfg: Cfg, sg, tg, G, F, E, ss=None, aux=None):
    """One tracking field (D42): candidate F'(x) = G(x), strict-min select.  Returns (F, E)."""
    sg = np.ascontiguousarray(sg, np.float32)
    tg = np.ascontiguousarray(tg, np.float32)
    h, w, _ = sg.shape
    G = np.ascontiguousarray(G, np.int32)
    F = np.array(F, np.int32, copy=True, order="C")
    E = np.array(E, np.float32, copy=True, order="C")
    ss_ = None if ss is None else np.ascontiguousarray(ss, np.float32)
    aux_ = None if aux is None else np.ascontiguousarray(aux, np.float32)
    cc = cfg.c()
    load().orc_track_field(C.byref(cc), h, w, _p(sg), _p(tg), None if ss_ is None else _p(ss_),
                           None if aux_ is None else _p(aux_), _p(G), _p(F), _p(E))
    return F, E
