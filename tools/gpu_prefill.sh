#!/bin/bash
# prefill: GPU tests of the batched path, compute-bound prefill bench, ncu launch list of one
# batched 16-token prefill (4 Mixtral-width layers, every expert resident)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "prefill or serialized or golden" > gpurun_out/pytest_prefill.log 2>&1; echo "pytest rc=$?" | tee -a gpurun_out/pytest_prefill.log; tail -2 gpurun_out/pytest_prefill.log
timeout 600 python tools/prefill_bench.py 4 1 4 16 64 > gpurun_out/prefill_bench.jsonl 2>&1
MOE_NCU_RANGE=1 timeout 600 /usr/local/cuda/bin/ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/prefill_launches.csv python tools/prefill_bench.py 4 16 > gpurun_out/prefill_ncu.log 2>&1
echo "ncu rc=$?"
