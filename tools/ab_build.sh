#!/bin/bash
# Builds A/B variants of libmoeb200.so with extra -D flags next to the product
# library, for microbenchmarks only (MOE_LIB_PATH=<variant> python tools/gemv_bench.py).
#   bash tools/ab_build.sh <tag> <nvcc -D flags...>
set -eu
ROOT=$(cd "$(dirname "$0")/.." && pwd)
tag=$1; shift
C=$ROOT/paper_2312_17238_b200/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -shared -lpthread "$@" -o "$ROOT/paper_2312_17238_b200/libmoeb200_ab_$tag.so" \
  $C/kernels.cu $C/tile.cu $C/engine.cu $C/store_sim.cu $C/blockio.cu
echo "built libmoeb200_ab_$tag.so"
