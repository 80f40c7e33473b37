#!/bin/bash
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=20000
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for v in 1 0; do
MOE_PF_W2=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_pf$v.log 2>&1; echo "pf=$v rc=$?"
tail -1 gpurun_out/bench_pf$v.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d['timeline']
print('value',d['value'],'ms',d['ms_per_step'])
print({k:v.get('median_us',v['avg_us']) for k,v in t['kernels'].items()}); p=t['phases_us']; print({k:p[k] for k in ('expert_up','expert_down','expert_down_epilogue','qkv','wo')})"
done
