#!/bin/bash
# full round-trip: smoke, gpu tests, C2/C3 bench, reference arm, launch list
bash tools/gpu_check2.sh
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/bench_ref.log | cut -c1-400
