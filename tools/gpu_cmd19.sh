#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/cta_trace.txt
MOE_CTA_TRACE_FILE=gpurun_out/cta_trace.txt timeout 300 python tools/gemv_bench.py > gpurun_out/gemv_bench.log 2>&1; echo "gemv rc=$?"
