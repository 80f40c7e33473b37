#!/bin/bash
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=20000
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for v in 1 0 1; do
MOE_BULK_EPI=$v timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_be$v.log 2>&1; echo "bulk=$v rc=$?"
tail -1 gpurun_out/bench_be$v.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d['timeline']
print('value',d['value'],'e2e',d['e2e']['value'],'ms',d['ms_per_step'])
print({k:v.get('median_us',v['avg_us']) for k,v in t['kernels'].items()}); p=t['phases_us']; print({k:p[k] for k in ('qkv_epilogue','wo_epilogue','expert_up_epilogue','expert_down_epilogue','combine_ln')})"
done
MOE_BULK_EPI=1 python tools/gemv_one.py 3 4096 14336 4 20; MOE_BULK_EPI=0 python tools/gemv_one.py 3 4096 14336 4 20
MOE_BULK_EPI=1 python tools/gemv_one.py 3 14336 4096 2 20; MOE_BULK_EPI=0 python tools/gemv_one.py 3 14336 4096 2 20
