#!/bin/bash
# One gpurun round trip: GPU tests, the bench (b200 arm) and the CPU reference
# arm.  Usage: gpurun --timeout 2400 -- 'bash tools/gpu_round.sh [tests] [bench] [ref]'
set -u
what=" ${*:-tests bench ref} "
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
if [[ $what == *" tests "* ]]; then
  timeout 1200 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?" | tee -a gpurun_out/pytest_gpu.log
fi
if [[ $what == *" bench "* ]]; then
  MOE_BENCH_VERBOSE=1 timeout 1200 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$?"; tail -c 600 gpurun_out/bench.json
fi
if [[ $what == *" ref "* ]]; then
  MOE_BENCH_VERBOSE=1 timeout 1700 python bench.py --impl reference ${REF_ARGS:---steps 20 --warmup 5} > gpurun_out/ref.json 2> gpurun_out/ref.err
  echo "ref rc=$?"; tail -c 600 gpurun_out/ref.json
fi
