#!/bin/bash
# Whole GPU suite, default bench line (config 2), launch list of one timed step, smoke.  Run under gpurun.
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 1500 python -m pytest tests/ -x -q -m gpu > gpurun_out/gpu_tests_$TAG.log 2>&1
tail -n 3 gpurun_out/gpu_tests_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -n 2 gpurun_out/smoke_$TAG.log
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err && cat gpurun_out/bench_$TAG.json | head -c 600; echo
[ -n "$NOLIST" ] || ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_list_$TAG.log 2>&1
