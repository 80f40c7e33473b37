#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/cta_trace2.txt
export MOE_CTA_TRACE_FILE=gpurun_out/cta_trace2.txt
python tools/gemv_one.py 3 14336 4096 2 20
python tools/gemv_one.py 3 4096 14336 4 20
python tools/gemv_one.py 4 4096 4096 3 20
python tools/gemv_one.py 4 4096 4096 1 20
python tools/cta_trace.py gpurun_out/cta_trace2.txt
