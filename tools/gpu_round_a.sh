#!/bin/bash
# r02 evidence batch: L1 peak microbenchmark, default bench line, world-2-on-one-GPU correctness runs, ncu
# captures of the non-dominant kernels.  Run under gpurun from the repo root.
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l1_peak_bench tools/l1_peak_bench.cu && \
    ./tools/l1_peak_bench > gpurun_out/l1_peak.json 2> gpurun_out/l1_peak.err
python bench.py > gpurun_out/bench_config2.json 2> gpurun_out/bench_config2.err
for wl in config1 config2 config3 config4; do
    timeout 900 python bench.py --gpus 2 --workload $wl --steps 2 --warmup 3 --check-single --no-cpu-baseline \
        > gpurun_out/bench_w2_$wl.json 2> gpurun_out/bench_w2_$wl.err
done
bash tools/profile_kernels.sh r02base "field0L0 tbarL0 gen0L1 gen1L1 gen2L1 gen3L1"
