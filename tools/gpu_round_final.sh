#!/bin/bash
# Final evidence batch on the current tree (run under gpurun from the repo root): GPU suite + smoke, default
# bench line (config 2), configs 3/4, world-2 check runs, ncu launch list of one timed config-2 step, ncu --set
# full of the dominant kernel.  Each ncu command runs only after its program exited 0 without ncu.
TAG=${TAG:-v10}
mkdir -p gpurun_out
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
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
    > gpurun_out/ncu_launches_$TAG.log 2>&1
python tools/prof_case.py 24 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_iter13 -s 2 -c 1 -f -o gpurun_out/full_$TAG \
    python tools/prof_case.py 24 > gpurun_out/ncu_full_$TAG.log 2>&1
ls gpurun_out | grep $TAG
