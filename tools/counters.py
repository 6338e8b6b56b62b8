"""Development aid: event counters of the fused level-0 kernel (library built with -DFB_COUNTERS by
tools/build_variant.sh cnt -DFB_COUNTERS, selected with FB_LIB).  One N-frame 512^2 blend.
usage: FB_LIB=paper_2311_09265_b200/libfb_vcnt.so python tools/counters.py N mode"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_09265_b200 as P  # noqa: E402
from synth import moving_texture  # noqa: E402

N, mode = int(sys.argv[1]), sys.argv[2]
g, s = moving_texture(N, 512, 512)
gd, sd = torch.from_numpy(g).cuda(), torch.from_numpy(s).cuda()
ctx = P.Context(0)
lib = ctx.lib
lib.fb_debug_counters.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 32)()
cfg = P.MatchCfg(loss=P.MEAN_ALIGN if mode == "accurate" else P.GUIDE_STYLE)
lib.fb_debug_counters(buf, 1)
ctx.fb_blend_window(cfg, P.DIRECT, gd, sd, 15)
torch.cuda.synchronize()
lib.fb_debug_counters(buf, 1)
c = list(buf)
for name, b in (("propagation", 0), ("random search", 8)):
    ev, s1, s2, full, win, same = c[b], c[b + 1], c[b + 2], c[b + 3], c[b + 4], c[b + 5]
    print(f"{name}: loss calls {ev:.4g}, PDE out after row 1 {s1 / max(ev, 1):.3f}, after row 3 {s2 / max(ev, 1):.3f}, "
          f"full {full / max(ev, 1):.3f}, wins {win / max(ev, 1):.4f}, incumbent-equal skipped {same:.4g}")
print(f"random search rejected by the patch-sum bound: {c[14]:.4g} "
      f"({c[14] / max(c[14] + c[8], 1):.3f} of candidates that differ from the incumbent)")
print(f"random search rejected by the partial + remainder bound after row 3: {c[21]:.4g} "
      f"({c[21] / max(c[8], 1):.3f} of its loss calls)")
