#!/bin/bash
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=20000
MOE_ROUTE_STAMPS=1 timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest(stamps) rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for v in 1 0 1; do
MOE_ROUTE_STAMPS=$v timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_st$v.log 2>&1; echo "stamps=$v rc=$?"
tail -1 gpurun_out/bench_st$v.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d['timeline']
print('value',d['value'],'e2e',d['e2e']['value'],'ms',d['ms_per_step'])
print({k:v.get('median_us',v['avg_us']) for k,v in t['kernels'].items()}); p=t['phases_us']; print({k:p[k] for k in ('tail','expert_up','expert_up_blk0')})"
done
