#!/bin/bash
# Experimental build of the library with extra -D flags into exp/ (A/B with FC_LIB=exp/<name>.so)
# usage: tools/exp_build.sh name -DFLAG=1 ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
mkdir -p "$ROOT/exp"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -shared \
  "$@" -o "$ROOT/exp/$name.so" "$ROOT/paper_1311_0089_b200/csrc/fc_engine.cu" -ldl
