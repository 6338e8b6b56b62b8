"""CPU oracle for FastBlend's hot path (arXiv 2311.09265).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It shares no code with the
CUDA product path in ``paper_2311_09265_b200``; the product never imports it.

The arithmetic lives in ``fb_oracle.c`` (plain C, FP32 in the paper's order, fmaf only where the
contract says fma).  ``oracle.py`` is argument marshalling.
"""
from .oracle import *  # noqa: F401,F403
