#!/bin/bash
# Development A/B: build the library with extra -D flags into paper_2311_09265_b200/libfb_v<name>.so
# (git-ignored, travels with gpurun); select it at run time with FB_LIB=<path>.
# usage: tools/build_variant.sh <name> [-DFOO=1 ...]
set -e
cd "$(dirname "$0")/.."
name=$1; shift
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false \
  -Xcompiler -fPIC -shared -Iinclude "$@" -o paper_2311_09265_b200/libfb_v$name.so \
  paper_2311_09265_b200/csrc/engine.cu paper_2311_09265_b200/csrc/kernels.cu
