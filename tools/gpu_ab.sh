#!/bin/bash
# Parity of the tests matching $1 (pytest -k), then A/B of option $2 at N=48 (accurate, balanced), then the whole
# GPU suite.  Run under gpurun from the repo root:  tools/gpu_ab.sh "<-k expr>" OPTION [values]
mkdir -p gpurun_out
K=$1; OPT=$2; VALS=${3:-0,1}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "$K" > gpurun_out/ab_tests.log 2>&1 || { tail -40 gpurun_out/ab_tests.log; exit 1; }
for mode in accurate balanced; do
    timeout 600 python tools/ab_env.py $OPT 48 $mode 2 $VALS > gpurun_out/ab_${OPT}_$mode.log 2>&1
done
[ -n "$NOSUITE" ] || timeout 1200 python -m pytest tests/ -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1
tail -n 3 gpurun_out/ab_tests.log; tail -n 3 gpurun_out/gpu_tests.log
cat gpurun_out/ab_${OPT}_*.log
