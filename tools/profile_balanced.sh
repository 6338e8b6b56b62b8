#!/bin/bash
# ncu --set full of the balanced-mode Ŝ refresh (k_aux_remap<2, SF8>), one instance, raw CSV for tools/ncu_summary.py
TAG=${1:-r02}
mkdir -p gpurun_out
python tools/prof_case.py 24 balanced > gpurun_out/prof_case_bal_$TAG.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k_aux_remap<\(int\)2, \(int\)0>" \
    -s 1 -c 1 -f -o gpurun_out/auxL0_$TAG python tools/prof_case.py 24 balanced > gpurun_out/ncu_auxL0_$TAG.log 2>&1
ncu -i gpurun_out/auxL0_$TAG.ncu-rep --page raw --csv > gpurun_out/auxL0_${TAG}_raw.csv 2>/dev/null
rm -f gpurun_out/auxL0_$TAG.ncu-rep
