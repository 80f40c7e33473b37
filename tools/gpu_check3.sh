#!/bin/bash
# tests (optionally a subset), bench, A/B GEMV microbench, prefill bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
AB_BENCH=${AB_BENCH:-} PREFILL=1 bash tools/gpu_ab.sh
