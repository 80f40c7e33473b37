#!/bin/bash
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=20000
timeout 300 python tools/gemv_bench.py > gpurun_out/gemv_bench.log 2>&1; echo "gemv rc=$?"
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
MOE_FAULTHANDLER=400 timeout 500 python bench.py > gpurun_out/bench_c2.log 2>&1; echo "bench c2 rc=$?"
MOE_FAULTHANDLER=400 timeout 500 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo "bench c3 rc=$?"
