#!/bin/bash
mkdir -p gpurun_out
for w in 2 3 4 6; do MOE_GEMV_WAVES=$w timeout 300 python tools/gemv_bench.py > gpurun_out/gemv_bench_w$w.log 2>&1; echo "gemv waves $w rc=$?"; done
