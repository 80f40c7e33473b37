#!/bin/bash
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=20000
timeout 300 python tools/debug_mixtral.py 2 2 2 > gpurun_out/dbg_c3.log 2>&1; echo "c3 rc=$?"
MOE_SERIAL_COPIES=1 MOE_NCU_RANGE=1 timeout 900 /usr/local/cuda/bin/ncu --profile-from-start off --set full --import-source on \
  -k "regex:k_tail|k_combine|k_attention128|k_embed" -c 4 -o gpurun_out/small -f \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_small.log 2>&1; echo "ncu small rc=$?"
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on -k regex:k_gemv -s 5 -c 1 -o gpurun_out/gemv3 -f python tools/gemv_one.py 3 4096 14336 4 8 > gpurun_out/ncu_gemv3.log 2>&1; echo "ncu gemv rc=$?"
timeout 600 python -m pytest tests/test_gpu_ep.py -q > gpurun_out/pytest_ep.log 2>&1; echo "ep rc=$?"; tail -3 gpurun_out/pytest_ep.log
