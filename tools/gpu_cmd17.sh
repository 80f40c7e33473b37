#!/bin/bash
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=20000
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; rc=$?; echo "smoke rc=$rc"
if [[ $rc != 0 ]]; then tail -5 gpurun_out/smoke.log; exit 1; fi
timeout 300 python tools/gemv_bench.py > gpurun_out/gemv_bench.log 2>&1; echo "gemv rc=$?"
timeout 900 python -m pytest tests -m gpu -q -x --timeout=240 --timeout-method=thread > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
MOE_FAULTHANDLER=300 timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench c2 rc=$?"
MOE_FAULTHANDLER=300 timeout 400 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo "bench c3 rc=$?"
