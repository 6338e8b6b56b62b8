#!/bin/bash
# One GPU call's worth of round evidence (run under gpurun from the repo root):
#   1. bench.py default line (config 2)                        -> gpurun_out/bench_$TAG.json
#   2. ncu launch list of one timed bench step (after warm-up)  -> gpurun_out/launches_$TAG.csv
#   3. ncu --set full of the dominant kernel (fused fields 1-3, level 0) on tools/prof_case.py 24
#                                                              -> gpurun_out/full_$TAG.ncu-rep
# Each ncu command runs only after its program exited 0 without ncu (the bench run above).
TAG=${1:-v7}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err || exit 1
python tools/prof_case.py 24 > /dev/null 2>&1 || exit 1
# bench --steps 1 --warmup 3: 3 x 136 warm-up launches, then the timed step's 136
ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 408 -c 136 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/ncu_launches_$TAG.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_iter13 -s 2 -c 1 -f -o gpurun_out/full_$TAG \
    python tools/prof_case.py 24 > gpurun_out/ncu_full_$TAG.log 2>&1
ls -la gpurun_out
