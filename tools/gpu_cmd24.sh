#!/bin/bash
# cluster threshold sweep on the C2 bench (timeline + value)
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=20000
timeout 600 python -m pytest tests/test_gpu_engine.py -q -x -k "mixtral or golden" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_quick.log
for cm in 1073741824 16 8; do
MOE_CLUSTER_MIN_S=$cm timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_cm$cm.log 2>&1; echo "cm=$cm rc=$?"
tail -1 gpurun_out/bench_cm$cm.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d['timeline']
print('value',d['value'],'ms',d['ms_per_step'])
print({k:v['avg_us'] for k,v in t['kernels'].items()}); print(t.get('phases_us'))"
done
