#!/bin/bash
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=20000
for v in 0 1; do
MOE_WO_LATE=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_wl$v.log 2>&1; echo "wolate=$v rc=$?"
tail -1 gpurun_out/bench_wl$v.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d['timeline']
print('value',d['value'],'ms',d['ms_per_step'])
print({k:v.get('median_us',v['avg_us']) for k,v in t['kernels'].items()}); p=t['phases_us']; print({k:p[k] for k in ('attention','wo','qkv')})"
done
MOE_FUSE_COMBINE=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_fc0.log 2>&1; echo "fc0 rc=$?"
tail -1 gpurun_out/bench_fc0.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d['timeline']
print('value',d['value'],'ms',d['ms_per_step'])
print({k:v.get('median_us',v['avg_us']) for k,v in t['kernels'].items()})"
