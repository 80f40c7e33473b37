#!/bin/bash
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=20000
timeout 300 python tools/gemv_bench.py > gpurun_out/gemv_bench.log 2>&1; echo "gemv rc=$?"
MOE_FAULTHANDLER=400 timeout 500 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench c2 rc=$?"
MOE_FAULTHANDLER=400 timeout 500 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo "bench c3 rc=$?"
timeout 600 python -m pytest tests/test_gpu_engine.py -q -k mixtral > gpurun_out/pytest_mixtral.log 2>&1; echo "mixtral rc=$?"; tail -2 gpurun_out/pytest_mixtral.log
