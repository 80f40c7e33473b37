#!/bin/bash
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=20000
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
python tools/gemv_bench.py > gpurun_out/gemv_bench.log 2>&1; grep '"pdl": 1' gpurun_out/gemv_bench.log | cut -c1-110
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench c2 rc=$?"
tail -1 gpurun_out/bench_c2.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d['timeline']
print('value',d['value'],'e2e',d['e2e']['value'],'ms',d['ms_per_step'], 'rl', d['roofline'].get('frac_timeline'))
print({k:v['median_us'] if 'median_us' in v else v['avg_us'] for k,v in t['kernels'].items()}); print(t.get('phases_us'))"
