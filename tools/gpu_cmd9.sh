#!/bin/bash
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=20000 MOE_BENCH_VERBOSE=1 MOE_FAULTHANDLER=150
MOE_COPY_TRACE=1 timeout 200 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b9_graph.log 2>&1; echo "graph rc=$?"
MOE_GRAPH=0 timeout 200 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b9_nograph.log 2>&1; echo "nograph rc=$?"
MOE_COPY_TRACE=1 timeout 200 python tools/debug_mixtral.py 2 2 2 > gpurun_out/b9_c3.log 2>&1; echo "c3 rc=$?"
