#!/bin/bash
mkdir -p gpurun_out
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on -k regex:k_gemv -s 5 -c 1 -o gpurun_out/gemv3b -f python tools/gemv_one.py 3 4096 14336 4 8 > gpurun_out/ncu_gemv3b.log 2>&1; echo "ncu rc=$?"
