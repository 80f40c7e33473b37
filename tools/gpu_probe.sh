#!/bin/bash
# GEMV probe: microbench (mma / CUDA-core layouts), GPU tests, optional ncu capture.
mkdir -p gpurun_out
timeout 300 python tools/gemv_bench.py > gpurun_out/gemv_mma.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
if [ -n "${NCU:-}" ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_mgemv -s 3 -c 1 \
  -o gpurun_out/gemv3_mma -f python tools/gemv_one.py 3 4096 14336 4 5 > gpurun_out/ncu.log 2>&1
fi
tail -3 gpurun_out/pytest_gpu.log
