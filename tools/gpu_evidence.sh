#!/bin/bash
# Round evidence batch: GPU suite, smoke, default bench line, bench lines of configs 3/4, world-2 runs on one GPU
# with the single-call check, launch list of one timed config-2 step.  Run under gpurun from the repo root.
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 1500 python -m pytest tests/ -x -q -m gpu > gpurun_out/gpu_tests_$TAG.log 2>&1; tail -n 2 gpurun_out/gpu_tests_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -n 1 gpurun_out/smoke_$TAG.log
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; head -c 300 gpurun_out/bench_$TAG.json; echo
for wl in config3 config4; do
    python bench.py --workload $wl --no-cpu-baseline > gpurun_out/bench_${wl}_$TAG.json 2> gpurun_out/bench_${wl}_$TAG.err
done
for wl in config1 config2 config3 config4; do
    timeout 900 python bench.py --gpus 2 --workload $wl --steps 2 --warmup 3 --check-single --no-cpu-baseline \
        > gpurun_out/w2_${wl}_$TAG.json 2> gpurun_out/w2_${wl}_$TAG.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_list_$TAG.log 2>&1
ls gpurun_out | grep $TAG
