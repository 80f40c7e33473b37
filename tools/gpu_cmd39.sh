#!/bin/bash
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=20000
timeout 300 python -m pytest tests/test_gpu_engine.py -q -x -k "teacher or mixtral_width_decode or golden" > gpurun_out/pytest_quick.log 2>&1; echo "quick rc=$?"; tail -1 gpurun_out/pytest_quick.log
for v in 1 0; do
MOE_PF_QKV=$v timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_pq$v.log 2>&1; echo "pfqkv=$v rc=$?"
tail -1 gpurun_out/bench_pq$v.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d['timeline']
print('value',d['value'],'ms',d['ms_per_step'])
print({k:v.get('median_us',v['avg_us']) for k,v in t['kernels'].items()}); p=t['phases_us']; print({k:p[k] for k in ('qkv','qkv_combine','expert_down','attention')})"
done
