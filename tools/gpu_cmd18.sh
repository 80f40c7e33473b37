#!/bin/bash
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=20000
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; rc=$?; echo "smoke rc=$rc"
if [[ $rc != 0 ]]; then tail -5 gpurun_out/smoke.log; exit 1; fi
for ms in 2 16 1000; do MOE_CLUSTER_MIN_S=$ms timeout 300 python tools/gemv_bench.py > gpurun_out/gemv_bench_$ms.log 2>&1; echo "gemv $ms rc=$?"; done
MOE_FAULTHANDLER=300 timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench c2 rc=$?"
