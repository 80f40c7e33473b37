#!/bin/bash
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=20000
MOE_DN_CLUSTER=4 timeout 900 python -m pytest tests/test_gpu_engine.py -q -x -k "mixtral or golden or teacher" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_quick.log
for v in 0 2 4; do
MOE_DN_CLUSTER=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_dc$v.log 2>&1; echo "dc=$v rc=$?"
tail -1 gpurun_out/bench_dc$v.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d['timeline']
print('value',d['value'],'ms',d['ms_per_step'])
print({k:v.get('median_us',v['avg_us']) for k,v in t['kernels'].items()}); p=t['phases_us']; print({k:p[k] for k in ('qkv','expert_down','expert_down_epilogue')})"
done
