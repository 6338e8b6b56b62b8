"""B200-native FastBlend hot path (arXiv 2311.09265): PatchMatch NNF estimation, remap/vote and the
sliding-window / keyframe blends as hand-written sm_100a CUDA kernels behind the C ABI in
include/fb.h.  This package is the product path: it never imports the CPU oracle."""
from . import fb  # noqa: F401
from .fb import (BASE, DIRECT, GUIDE_STYLE, INIT_IDENTITY, INIT_RANDOM, MEAN_ALIGN, PAIRWISE, SYMBOLS, TREE, Context,  # noqa: F401
                 FBError, MatchCfg, blend_window_e2e, load_library)
