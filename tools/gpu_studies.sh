#!/bin/bash
# §8(f)2 trace-driven sweep + §8(f)4 Table-2 ablation (one gpurun call)
mkdir -p gpurun_out
if [[ " ${*:-trace ablation} " == *" trace "* ]]; then
  timeout 1500 python tools/trace_sweep.py --config c3 --out gpurun_out/trace_sweep_c3 > gpurun_out/trace_sweep.log 2>&1
  echo "trace_sweep rc=$?"; tail -25 gpurun_out/trace_sweep.log
fi
if [[ " ${*:-trace ablation} " == *" ablation "* ]]; then
  timeout 2400 python tools/ablation.py --out gpurun_out/ablation.md > gpurun_out/ablation.log 2>&1
  echo "ablation rc=$?"; tail -20 gpurun_out/ablation.md
fi
