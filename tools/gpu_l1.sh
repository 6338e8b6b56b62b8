#!/bin/bash
# Level-1 fast path (SF10 + TF10 through the mid / fused kernels): parity first, then A/B timings, then the
# whole GPU suite.  Run under gpurun from the repo root.
mkdir -p gpurun_out
python -c "from paper_2311_09265_b200 import build as b; b.build_library()"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "level1" > gpurun_out/l1_tests.log 2>&1 || { tail -30 gpurun_out/l1_tests.log; exit 1; }
timeout 600 python tools/ab_env.py L1_FAST 48 accurate 2 > gpurun_out/ab_l1_accurate.log 2>&1
timeout 600 python tools/ab_env.py L1_FAST 48 balanced 2 > gpurun_out/ab_l1_balanced.log 2>&1
timeout 1200 python -m pytest tests/ -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/l1_tests.log gpurun_out/gpu_tests.log
cat gpurun_out/ab_l1_*.log
