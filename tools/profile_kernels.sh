#!/bin/bash
# ncu --set full captures of the non-dominant kernels of a config-2-shaped accurate blend (tools/prof_case.py),
# one kernel instance each, exported as raw CSV for tools/ncu_summary.py.  Run under gpurun from the repo root:
#   tools/profile_kernels.sh TAG ["name1 name2 ..."]
# Each capture only after prof_case.py itself exited 0 without ncu.
TAG=${1:-r02}
ONLY=${2:-}
mkdir -p gpurun_out
python tools/prof_case.py 24 > gpurun_out/prof_case_$TAG.log 2>&1 || exit 1
cap() {  # name regex skip   (ONLY = space-separated names to capture; empty = all)
    if [ -n "$ONLY" ] && [[ " $ONLY " != *" $1 "* ]]; then return; fi
    ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$2" -s "$3" -c 1 -f \
        -o gpurun_out/${1}_$TAG python tools/prof_case.py 24 > gpurun_out/ncu_${1}_$TAG.log 2>&1
    ncu -i gpurun_out/${1}_$TAG.ncu-rep --page raw --csv > gpurun_out/${1}_${TAG}_raw.csv 2>/dev/null
    # per-source-line stall samples (needs -lineinfo): KEEP_SRC=1
    [ -z "$KEEP_SRC" ] || ncu -i gpurun_out/${1}_$TAG.ncu-rep --page source --csv > gpurun_out/${1}_${TAG}_src.csv 2>/dev/null
    [ -n "$KEEP_REP" ] || rm -f gpurun_out/${1}_$TAG.ncu-rep  # gpurun copies back <= 64 MiB
}
# demangled names read e.g. "void fbk::k_field_gen<(int)2, (bool)1, (int)0, (int)4, (bool)0>(fbk::FieldArgs)"
cap field0L0 "k_field_mid" 1
cap tbarL0 "k_combine<\\(int\\)2, \\(int\\)2>" 1
cap gen0L1 "k_field_gen<\\(int\\)2, \\(bool\\)1, \\(int\\)0, \\(int\\)4" 1
cap gen1L1 "k_field_gen<\\(int\\)2, \\(bool\\)1, \\(int\\)1, \\(int\\)4" 1
cap gen2L1 "k_field_gen<\\(int\\)2, \\(bool\\)1, \\(int\\)2, \\(int\\)4" 1
cap gen3L1 "k_field_gen<\\(int\\)2, \\(bool\\)1, \\(int\\)3, \\(int\\)4" 1
cap field123L0 "k_iter13_fast" 1
cap tbarL1 "k_combine<\\(int\\)2, \\(int\\)3>" 15  # level 1 (coarse-to-fine: levels 4, 3, 2 first)
cap combine "k_combine<\\(int\\)2, \\(int\\)1>" 0
cap gen3L2 "k_field_gen<\\(int\\)2, \\(bool\\)1, \\(int\\)3, \\(int\\)2" 10  # level 2 (after levels 4, 3)
ls -la gpurun_out
