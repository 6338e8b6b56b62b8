#!/bin/bash
# cost split of the accurate N=48 blend + ncu full of the fused level-0 kernel (tools/profile_kernels.sh)
mkdir -p gpurun_out
timeout 900 python tools/cost_split.py 48 accurate "default:" "nobound:opt.SUM_BOUND=0" "rs1:rs_steps=1,rs_radius0=1" \
    "rs1_nob:rs_steps=1,rs_radius0=1,opt.SUM_BOUND=0" "rs5:rs_steps=5" "alpha0:alpha=0" > gpurun_out/split.log 2>&1
cat gpurun_out/split.log
bash tools/profile_kernels.sh ${TAG:-r02csb} "field123L0"
