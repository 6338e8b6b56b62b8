"""Thin Python binding of the C ABI in include/fb.h (argument marshalling only).

Every step of the hot path runs in libfastblend.so's sm_100a kernels; PyTorch provides device memory,
streams and host staging.  There is no fallback: if the library or a CUDA device is missing, the calls
raise.  Function names follow the C entry points (fb_build_pyramid, fb_nnf_estimate, fb_remap,
fb_blend_window, fb_interpolate_keyframes).
"""
from __future__ import annotations

import contextlib
import ctypes as C
import os
from dataclasses import dataclass

import torch

from . import build as _build

BASE, GUIDE_STYLE, MEAN_ALIGN, PAIRWISE = 0, 1, 2, 3
DIRECT, TREE = 0, 1
INIT_RANDOM, INIT_IDENTITY = 0, 1
OP_NNF, OP_BLEND_DIRECT, OP_BLEND_TREE, OP_INTERPOLATE = 0, 1, 2, 3
OPT_FUSED_ITER, OPT_FUSE13, OPT_PHASE0_MID, OPT_TGT_REG_ROWS, OPT_L1_FAST, OPT_SUM_BOUND, OPT_P3_FUSED = 0, 1, 2, 3, 4, 5, 6
OPT_TAIL_BOUND = 7
TAG_DIRECT, TAG_TREE_BUILD_F, TAG_TREE_QUERY_F, TAG_TREE_BUILD_R, TAG_TREE_QUERY_R, TAG_INTERP, TAG_API = range(7)

STATUS = {0: "FB_OK", 1: "FB_ERR_INVALID_ARG", 2: "FB_ERR_SHAPE", 3: "FB_ERR_CUDA", 4: "FB_ERR_NCCL",
          5: "FB_ERR_WORKSPACE", 6: "FB_ERR_UNSUPPORTED"}

SYMBOLS = ["fb_ctx_create", "fb_ctx_destroy", "fb_last_error", "fb_set_workspace", "fb_set_max_batch_pairs",
           "fb_workspace_size", "fb_workspace_size_range", "fb_launch_count", "fb_set_option", "fb_pyramid_elems", "fb_build_pyramid", "fb_nnf_estimate",
           "fb_remap", "fb_blend_window", "fb_blend_window_range", "fb_interpolate_keyframes", "fb_profile_enable",
           "fb_profile_read", "fb_profile_reset", "fb_tree_cell_texels", "fb_tree_build_cells", "fb_tree_query",
           "fb_interpolate_keyframes_range"]


class FBError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class _Cfg(C.Structure):
    _fields_ = [("patch_radius", C.c_int32), ("levels", C.c_int32), ("iters_per_level", C.c_int32),
                ("rs_radius0", C.c_int32), ("rs_steps", C.c_int32), ("alpha", C.c_float),
                ("loss", C.c_int32), ("init", C.c_int32), ("seed", C.c_uint64), ("prop_scales", C.c_int32),
                ("tracking", C.c_int32)]


class _Stats(C.Structure):
    _fields_ = [("nnf_pairs", C.c_uint64), ("candidate_evals", C.c_uint64), ("remap_pixels", C.c_uint64)]

    def as_dict(self):
        return {"nnf_pairs": int(self.nnf_pairs), "candidate_evals": int(self.candidate_evals),
                "remap_pixels": int(self.remap_pixels)}


class _Prof(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_uint64), ("ms", C.c_double), ("work", C.c_uint64)]


class _Key(C.Structure):
    _fields_ = [("src_id", C.c_int32), ("tgt_id", C.c_int32), ("task_tag", C.c_int32)]


@dataclass
class MatchCfg:
    """fb_match_cfg.  Defaults: "patch 5" (p=2), auto pyramid, n=5, full-image random search,
    alpha=10, Philox seed 1, unit-step propagation (D1, D6, D13-D15, D41)."""
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


def load_library(build_if_missing: bool = True):
    """Loads libfastblend.so (building it in-tree with nvcc if needed).  Raises if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("FB_LIB", _build.LIB)  # FB_LIB: development A/B of alternative builds
    if path == _build.LIB and build_if_missing and _build.needs_build():
        _build.build_library()
    if not os.path.exists(path):
        raise RuntimeError(f"libfastblend.so not found at {path}; run __graft_entry__.build()")
    lib = C.CDLL(path)
    P, V = C.POINTER, C.c_void_p
    lib.fb_ctx_create.argtypes = [C.c_int, V, P(V)]
    lib.fb_ctx_destroy.argtypes = [V]
    lib.fb_ctx_destroy.restype = None
    lib.fb_last_error.argtypes = [V]
    lib.fb_last_error.restype = C.c_char_p
    lib.fb_set_workspace.argtypes = [V, V, C.c_size_t]
    lib.fb_set_max_batch_pairs.argtypes = [V, C.c_int64]
    lib.fb_workspace_size.argtypes = [V, C.c_int, P(_Cfg), C.c_int, C.c_int, C.c_int, C.c_int]
    lib.fb_workspace_size.restype = C.c_size_t
    lib.fb_workspace_size_range.argtypes = [V, C.c_int, P(_Cfg)] + [C.c_int] * 8
    lib.fb_workspace_size_range.restype = C.c_size_t
    lib.fb_set_option.argtypes = [V, C.c_int, C.c_int]
    lib.fb_launch_count.argtypes = [V]
    lib.fb_launch_count.restype = C.c_uint64
    lib.fb_pyramid_elems.argtypes = [C.c_int] * 4
    lib.fb_pyramid_elems.restype = C.c_size_t
    lib.fb_build_pyramid.argtypes = [V, V, C.c_int, C.c_int, C.c_int, C.c_int, V]
    lib.fb_nnf_estimate.argtypes = [V, P(_Cfg), C.c_int, C.c_int, C.c_int, V, V, V, V, V, V, V, V, V, P(_Stats)]
    lib.fb_remap.argtypes = [V, C.c_int, C.c_int, C.c_int, C.c_int, V, V, V]
    lib.fb_blend_window.argtypes = [V, P(_Cfg), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, V, V, V, P(_Stats)]
    lib.fb_blend_window_range.argtypes = [V, P(_Cfg), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                          V, V, C.c_int, C.c_int, V, P(_Stats)]
    lib.fb_interpolate_keyframes.argtypes = [V, P(_Cfg), C.c_int, C.c_int, C.c_int, V, C.c_int, V, V, V, P(_Stats)]
    lib.fb_interpolate_keyframes_range.argtypes = [V, P(_Cfg)] + [C.c_int] * 5 + [V, C.c_int, V, V, V, V, P(_Stats),
                                                                                P(C.c_size_t)]
    lib.fb_tree_cell_texels.argtypes = [P(_Cfg), C.c_int, C.c_int]
    lib.fb_tree_cell_texels.restype = C.c_size_t
    lib.fb_tree_build_cells.argtypes = [V, P(_Cfg)] + [C.c_int] * 5 + [V, V, C.c_int, V, V, P(_Stats), P(C.c_size_t)]
    lib.fb_tree_query.argtypes = [V, P(_Cfg)] + [C.c_int] * 6 + [V, V, C.c_int, C.c_int, C.c_int, V, V, V, P(_Stats),
                                                                P(C.c_size_t)]
    lib.fb_profile_enable.argtypes = [V, C.c_int]
    lib.fb_profile_read.argtypes = [V, P(_Prof), C.c_int]
    lib.fb_profile_read.restype = C.c_int
    lib.fb_profile_reset.argtypes = [V]
    lib.fb_profile_reset.restype = None
    for fn in ("fb_set_option", "fb_profile_enable", "fb_ctx_create", "fb_set_workspace", "fb_set_max_batch_pairs", "fb_build_pyramid", "fb_nnf_estimate",
               "fb_remap", "fb_blend_window", "fb_blend_window_range", "fb_interpolate_keyframes"):
        getattr(lib, fn).restype = C.c_int
    _lib = lib
    return lib


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _dev(t: torch.Tensor, device, dtype) -> torch.Tensor:
    if t.dtype != dtype:
        raise TypeError(f"expected {dtype}, got {t.dtype}")
    if t.device != device:
        t = t.to(device, non_blocking=True)
    return t.contiguous()


class Context:
    """An fb_ctx bound to one CUDA device and the torch stream current at creation; owns a growable
    workspace tensor (the library itself never allocates device memory)."""

    def __init__(self, device: int | torch.device = 0, stream: torch.cuda.Stream | None = None,
                 max_batch_pairs: int = 0):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2311_09265_b200 needs a CUDA device (no CPU fallback)")
        self.lib = load_library()
        self.device = torch.device("cuda", torch.device(device).index if not isinstance(device, int) else device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = C.c_void_p()
        self._check(self.lib.fb_ctx_create(self.device.index, C.c_void_p(self.stream.cuda_stream), C.byref(h)), h)
        self.h = h
        self.ws = None
        if max_batch_pairs:
            self.set_max_batch_pairs(max_batch_pairs)

    @contextlib.contextmanager
    def _ordered(self):
        """Orders the context stream after the caller's current stream (inputs copied, outputs and workspace
        allocated there) and the current stream after the context stream (outputs ready, buffers safe to free
        or reuse there).  A no-op when the context enqueues on the current stream."""
        cur = torch.cuda.current_stream(self.device)
        if cur == self.stream:
            yield
            return
        self.stream.wait_stream(cur)
        try:
            yield
        finally:
            cur.wait_stream(self.stream)

    def _run(self, status_fn, *args):
        with self._ordered():
            status = status_fn(self.h, *args)
        self._check(status)

    def _check(self, status: int, h=None):
        if status != 0:
            msg = self.lib.fb_last_error(h if h is not None else self.h)
            raise FBError(status, msg.decode() if msg else "")

    def close(self):
        if getattr(self, "h", None):
            self.lib.fb_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_max_batch_pairs(self, n: int):
        self._check(self.lib.fb_set_max_batch_pairs(self.h, int(n)))

    def set_option(self, option: int, value: int):
        """fb_set_option: an equivalent kernel schedule (OPT_*; results are bit-identical for every value)."""
        self._check(self.lib.fb_set_option(self.h, int(option), int(value)))

    def launch_count(self) -> int:
        return int(self.lib.fb_launch_count(self.h))

    def profile_enable(self, on: bool = True):
        self._check(self.lib.fb_profile_enable(self.h, int(bool(on))))

    def profile_reset(self):
        self.lib.fb_profile_reset(self.h)

    def profile_read(self) -> dict:
        """{kernel class: {"launches", "ms", "work"}} over the launches since the last reset."""
        n = self.lib.fb_profile_read(self.h, None, 0)
        arr = (_Prof * max(n, 1))()
        n = self.lib.fb_profile_read(self.h, arr, n)
        return {arr[i].name.decode(): {"launches": int(arr[i].launches), "ms": float(arr[i].ms),
                                       "work": int(arr[i].work)} for i in range(n)}

    def workspace_size(self, op: int, cfg: MatchCfg, n: int, H: int, W: int, M: int = 0) -> int:
        c = cfg.c()
        return int(self.lib.fb_workspace_size(self.h, op, C.byref(c), n, H, W, M))

    def ensure_workspace(self, nbytes: int):
        if nbytes <= 0:  # invalid arguments: the entry point itself reports the precise status
            return
        if self.ws is None or self.ws.numel() < nbytes:
            self.ws = None  # freed on its allocation stream, which waited for this context's last call (_ordered)
            self.ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            if self.stream != torch.cuda.current_stream(self.device):
                self.ws.record_stream(self.stream)
            self._check(self.lib.fb_set_workspace(self.h, C.c_void_p(self.ws.data_ptr()), self.ws.numel()))

    # ------------------------------------------------------------------------------ entry points
    def fb_build_pyramid(self, frames: torch.Tensor, levels: int) -> torch.Tensor:
        frames = _dev(frames, self.device, torch.uint8)
        B, H, W, _ = frames.shape
        n = int(self.lib.fb_pyramid_elems(B, H, W, levels))
        out = torch.empty(n, dtype=torch.float32, device=self.device)
        self._run(self.lib.fb_build_pyramid, _ptr(frames), B, H, W, levels, _ptr(out))
        return out.view(B, -1, 4)

    def fb_nnf_estimate(self, cfg: MatchCfg, src_guide, tgt_guide, src_style=None, tgt_style=None, group=None,
                        pair_keys=None, want_err: bool = True, want_remap: bool = True):
        """Returns (nnf int32 [B,H,W,2], err float [B,H,W] | None, remapped float [B,H,W,3] | None, stats)."""
        sg = _dev(src_guide, self.device, torch.uint8)
        tg = _dev(tgt_guide, self.device, torch.uint8)
        ss = None if src_style is None else _dev(src_style, self.device, torch.uint8)
        ts = None if tgt_style is None else _dev(tgt_style, self.device, torch.uint8)
        B, H, W, _ = sg.shape
        keys = (_Key * B)(*[_Key(*k) for k in (pair_keys or [(0, 0, TAG_API)] * B)])
        grp = None
        if group is not None:
            grp = (C.c_int32 * B)(*[int(x) for x in group])
        self.ensure_workspace(self.workspace_size(OP_NNF, cfg, B, H, W))
        nnf = torch.empty((B, H, W, 2), dtype=torch.int32, device=self.device)
        err = torch.empty((B, H, W), dtype=torch.float32, device=self.device) if want_err else None
        rem = torch.empty((B, H, W, 3), dtype=torch.float32, device=self.device) if want_remap and ss is not None else None
        st = _Stats()
        c = cfg.c()
        self._run(self.lib.fb_nnf_estimate, C.byref(c), B, H, W, _ptr(sg), _ptr(tg), _ptr(ss), _ptr(ts),
                                             grp, keys, _ptr(nnf), _ptr(err), _ptr(rem), C.byref(st))
        return nnf, err, rem, st.as_dict()

    def fb_remap(self, src: torch.Tensor, nnf: torch.Tensor, p: int) -> torch.Tensor:
        src = _dev(src, self.device, torch.float32)
        nnf = _dev(nnf, self.device, torch.int32)
        B, H, W, _ = src.shape
        out = torch.empty_like(src)
        self._run(self.lib.fb_remap, B, H, W, p, _ptr(src), _ptr(nnf), _ptr(out))
        return out

    def fb_blend_window(self, cfg: MatchCfg, schedule: int, guide, style, M: int, out: torch.Tensor | None = None):
        """Window blend of the whole video: returns (out float [N,H,W,3] in 8-bit units, stats)."""
        g = _dev(guide, self.device, torch.uint8)
        s = _dev(style, self.device, torch.uint8)
        N, H, W, _ = g.shape
        op = OP_BLEND_TREE if schedule == TREE else OP_BLEND_DIRECT
        self.ensure_workspace(self.workspace_size(op, cfg, N, H, W, M))
        if out is None:
            out = torch.empty((N, H, W, 3), dtype=torch.float32, device=self.device)
        st = _Stats()
        c = cfg.c()
        self._run(self.lib.fb_blend_window, C.byref(c), schedule, N, H, W, M, _ptr(g), _ptr(s), _ptr(out),
                                             C.byref(st))
        return out, st.as_dict()

    # ---- sharded tree schedule with cell exchange (include/fb.h) -------------------------
    def tree_cell_texels(self, cfg: MatchCfg, H: int, W: int) -> int:
        c = cfg.c()
        n = int(self.lib.fb_tree_cell_texels(C.byref(c), H, W))
        if n == 0:
            raise FBError(1, "invalid configuration for the frame size")
        return n

    @staticmethod
    def _cells(cells):
        flat = [int(x) for cell in cells for x in cell]
        return (C.c_int32 * max(len(flat), 1))(*flat), len(cells)

    def fb_tree_build_cells(self, cfg: MatchCfg, N_total: int, f0: int, guide, style, cells):
        """Builds the cells [(orient, j, L), ...] from local frames f0..f0+N-1: (float32 [n, texels, 4], stats)."""
        g = _dev(guide, self.device, torch.uint8)
        s = _dev(style, self.device, torch.uint8)
        N, H, W, _ = g.shape
        arr, n = self._cells(cells)
        c = cfg.c()
        need = C.c_size_t(0)
        self._run(self.lib.fb_tree_build_cells, C.byref(c), N_total, f0, N, H, W, _ptr(g), _ptr(s), n, arr,
                                                  None, None, C.byref(need))
        self.ensure_workspace(int(need.value))
        out = torch.empty((n, self.tree_cell_texels(cfg, H, W), 4), dtype=torch.float32, device=self.device)
        st = _Stats()
        self._run(self.lib.fb_tree_build_cells, C.byref(c), N_total, f0, N, H, W, _ptr(g), _ptr(s), n, arr,
                                                  _ptr(out), C.byref(st), None)
        return out, st.as_dict()

    def fb_tree_query(self, cfg: MatchCfg, N_total: int, f0: int, guide, style, M: int, t0: int, t1: int, cells,
                      cell_tensors, out: torch.Tensor | None = None):
        """Targets [t0, t1) from local frames plus cells (list of (orient, j, L)) whose pyramids are the
        matching entries of cell_tensors (a list of [texels, 4] tensors or one [n, texels, 4] tensor)."""
        g = _dev(guide, self.device, torch.uint8)
        s = _dev(style, self.device, torch.uint8)
        N, H, W, _ = g.shape
        arr, n = self._cells(cells)
        tens = [t.contiguous() for t in cell_tensors] if n else []
        for t in tens:
            if t.device != self.device or t.dtype != torch.float32:
                raise ValueError("cell tensors must be float32 on the context device")
        ptrs = (C.c_void_p * max(n, 1))(*[t.data_ptr() for t in tens])
        c = cfg.c()
        need = C.c_size_t(0)
        self._run(self.lib.fb_tree_query, C.byref(c), N_total, f0, N, H, W, M, _ptr(g), _ptr(s), t0, t1, n,
                                            arr, ptrs, None, None, C.byref(need))
        self.ensure_workspace(int(need.value))
        if out is None:
            out = torch.empty((t1 - t0, H, W, 3), dtype=torch.float32, device=self.device)
        st = _Stats()
        self._run(self.lib.fb_tree_query, C.byref(c), N_total, f0, N, H, W, M, _ptr(g), _ptr(s), t0, t1, n,
                                            arr, ptrs, _ptr(out), C.byref(st), None)
        return out, st.as_dict()

    def fb_blend_window_range(self, cfg: MatchCfg, schedule: int, N_total: int, f0: int, guide, style, M: int,
                              t0: int, t1: int, out: torch.Tensor | None = None):
        """Shard form: guide/style hold frames f0..f0+N-1 of an N_total-frame video; writes targets [t0,t1)."""
        g = _dev(guide, self.device, torch.uint8)
        s = _dev(style, self.device, torch.uint8)
        N, H, W, _ = g.shape
        c0 = cfg.c()
        self.ensure_workspace(int(self.lib.fb_workspace_size_range(self.h, schedule, C.byref(c0), N_total, f0, N, H, W, M,
                                                                   t0, t1)))
        if out is None:
            out = torch.empty((t1 - t0, H, W, 3), dtype=torch.float32, device=self.device)
        st = _Stats()
        c = cfg.c()
        self._run(self.lib.fb_blend_window_range, C.byref(c), schedule, N_total, f0, N, H, W, M, _ptr(g),
                                                    _ptr(s), t0, t1, _ptr(out), C.byref(st))
        return out, st.as_dict()

    def fb_interpolate_keyframes(self, cfg: MatchCfg, guide, key_index, key_style, out: torch.Tensor | None = None):
        g = _dev(guide, self.device, torch.uint8)
        ks = _dev(key_style, self.device, torch.uint8)
        N, H, W, _ = g.shape
        keys = [int(k) for k in key_index]
        K = len(keys)
        self.ensure_workspace(self.workspace_size(OP_INTERPOLATE, cfg, N, H, W, max(K, 1)))
        if out is None:
            out = torch.empty((N, H, W, 3), dtype=torch.float32, device=self.device)
        ki = (C.c_int32 * max(K, 1))(*keys)
        st = _Stats()
        c = cfg.c()
        self._run(self.lib.fb_interpolate_keyframes, C.byref(c), N, H, W, _ptr(g), K, ki, _ptr(ks), _ptr(out),
                                                      C.byref(st))
        return out, st.as_dict()


    def fb_interpolate_keyframes_range(self, cfg: MatchCfg, N: int, t0: int, t1: int, guide, key_index, key_guide,
                                       key_style, out: torch.Tensor | None = None):
        """Frames [t0, t1) of the interpolation (guide holds frames t0..t1-1; key_guide/key_style the K keys)."""
        g = _dev(guide, self.device, torch.uint8)
        kg = _dev(key_guide, self.device, torch.uint8)
        ks = _dev(key_style, self.device, torch.uint8)
        _, H, W, _ = g.shape
        keys = [int(k) for k in key_index]
        K = len(keys)
        ki = (C.c_int32 * max(K, 1))(*keys)
        c = cfg.c()
        need = C.c_size_t(0)
        self._run(self.lib.fb_interpolate_keyframes_range, C.byref(c), N, H, W, t0, t1, _ptr(g), K, ki, _ptr(kg),
                                                            _ptr(ks), None, None, C.byref(need))
        self.ensure_workspace(int(need.value))
        if out is None:
            out = torch.empty((t1 - t0, H, W, 3), dtype=torch.float32, device=self.device)
        st = _Stats()
        self._run(self.lib.fb_interpolate_keyframes_range, C.byref(c), N, H, W, t0, t1, _ptr(g), K, ki, _ptr(kg),
                                                            _ptr(ks), _ptr(out), C.byref(st), None)
        return out, st.as_dict()


def blend_window_e2e(ctx: Context, cfg: MatchCfg, schedule: int, guide_host: torch.Tensor, style_host: torch.Tensor,
                     M: int, out_host: torch.Tensor | None = None):
    """End-to-end public call on HOST tensors: H2D copies of the frames, the blend, D2H of the result."""
    out, st = ctx.fb_blend_window(cfg, schedule, guide_host, style_host, M)
    if out_host is None:
        out_host = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
    out_host.copy_(out, non_blocking=True)
    return out_host, st
