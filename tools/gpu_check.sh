#!/bin/bash
# One gpurun round trip: GPU parity tests, smoke, bench, ncu launch list and one
# full capture of the top kernel.  Usage (from this container):
#   gpurun --timeout 1800 -- 'bash tools/gpu_check.sh [tests|bench|ncu|all]'
set -u
what=" ${*:-all} "
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,pcie.link.gen.current,pcie.link.width.current --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import torch; print(torch.cuda.get_device_name(0))" >> gpurun_out/gpu.txt 2>&1
if [[ $what == *" all "* || $what == *" tests "* ]]; then
  timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; rc=$?; echo "smoke rc=$rc" | tee -a gpurun_out/smoke.log
  if [[ $rc != 0 ]]; then echo "smoke failed: stopping"; exit 1; fi
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a gpurun_out/pytest_gpu.log
fi
if [[ $what == *" all "* || $what == *" bench "* ]]; then
  timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" | tee -a gpurun_out/bench.log
  tail -1 gpurun_out/bench.log
fi
if [[ $what == *" all "* || $what == *" ncu "* ]]; then
  NCU=/usr/local/cuda/bin/ncu
  MOE_SERIAL_COPIES=1 MOE_NCU_RANGE=1 timeout 900 $NCU --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
     --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/ncu_launch.log 2>&1
  echo "ncu launches rc=$?"
  MOE_SERIAL_COPIES=1 MOE_NCU_RANGE=1 timeout 900 $NCU --profile-from-start off --set full --clock-control none --import-source on \
     -k regex:${NCU_KERNEL:-k_gemv} -s ${NCU_SKIP:-2} -c ${NCU_COUNT:-3} -o gpurun_out/prof -f \
     python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/ncu_full.log 2>&1
  echo "ncu full rc=$?"
fi
if [[ $what == *" mb "* ]]; then
  (cd tools && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb microbench.cu -lcuda && timeout 300 /tmp/mb) > gpurun_out/microbench.log 2>&1
  echo "microbench rc=$?"
fi
