#!/bin/bash
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=20000
for v in 0 1; do
MOE_COMB_HOLD=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_hold$v.log 2>&1; echo "hold=$v rc=$?"
tail -1 gpurun_out/bench_hold$v.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d['timeline']
print('value',d['value'],'ms',d['ms_per_step'])
print({k:v.get('median_us',v['avg_us']) for k,v in t['kernels'].items()}); p=t['phases_us']; print({k:p[k] for k in ('qkv','qkv_combine')})"
done
