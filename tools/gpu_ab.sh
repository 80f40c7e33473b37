#!/bin/bash
# A/B round trip: GEMV microbench for the product library and each A/B build
# (tools/ab_build.sh), the compute-bound prefill bench, optional bench lines.
mkdir -p gpurun_out
timeout 300 python tools/gemv_bench.py > gpurun_out/gemv_base.jsonl 2>&1
for lib in paper_2312_17238_b200/libmoeb200_ab_*.so; do
  tag=$(basename $lib .so); tag=${tag#libmoeb200_ab_}
  MOE_LIB_PATH=$PWD/$lib timeout 300 python tools/gemv_bench.py > gpurun_out/gemv_$tag.jsonl 2>&1
  if [ -n "${AB_BENCH:-}" ]; then
    MOE_LIB_PATH=$PWD/$lib timeout 600 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > gpurun_out/bench_$tag.json 2>gpurun_out/bench_$tag.err
  fi
done
if [ -n "${AB_BENCH:-}" ]; then
  timeout 600 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > gpurun_out/bench_base.json 2>gpurun_out/bench_base.err
fi
if [ -n "${PREFILL:-}" ]; then
  timeout 600 python tools/prefill_bench.py 4 1 4 16 64 > gpurun_out/prefill_bench.jsonl 2>&1
fi
