#!/bin/bash
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=20000
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
MOE_FAULTHANDLER=400 timeout 500 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench c2 rc=$?"
