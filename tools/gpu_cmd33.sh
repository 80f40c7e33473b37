#!/bin/bash
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=20000
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench c2 rc=$?"
tail -1 gpurun_out/bench_c2.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d['timeline']
print('value',d['value'],'e2e',d['e2e']['value'],'ms',d['ms_per_step'])
print({k:v.get('median_us',v['avg_us']) for k,v in t['kernels'].items()}); p=t['phases_us']; print({k:p[k] for k in ('tail','tail_thread0')})"
python tools/gemv_bench.py > gpurun_out/gemv_bench.log 2>&1; grep '"pdl": 1' gpurun_out/gemv_bench.log | cut -c1-100
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:k_gemv -s 5 -c 1 -o gpurun_out/gemv3_up -f python tools/gemv_one.py 3 4096 14336 4 8 > gpurun_out/ncu_up.log 2>&1; echo "ncu up rc=$?"
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:k_gemv -s 5 -c 1 -o gpurun_out/gemv3_down -f python tools/gemv_one.py 3 14336 4096 2 8 > gpurun_out/ncu_down.log 2>&1; echo "ncu down rc=$?"
