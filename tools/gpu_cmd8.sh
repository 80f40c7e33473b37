#!/bin/bash
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=15000
MOE_COPY_TRACE=1 timeout 300 python tools/debug_mixtral.py 2 2 2 > gpurun_out/dbg_c3_trace.log 2>&1; echo "c3 trace rc=$?"
timeout 600 python -m pytest tests/test_gpu_ep.py -x -q > gpurun_out/pytest_ep.log 2>&1; echo "ep rc=$?"; tail -3 gpurun_out/pytest_ep.log
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on -k regex:k_gemv -s 5 -c 1 -o gpurun_out/gemv3 -f python tools/gemv_one.py 3 4096 14336 4 8 > gpurun_out/ncu_gemv3.log 2>&1; echo "ncu rc=$?"
