#!/bin/bash
# all-hit compute time (k=8) vs C2, and a short copy trace
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=20000
for k in 8 4; do
timeout 600 python bench.py --no-cpu-baseline --no-e2e --k $k > gpurun_out/bench_k$k.log 2>&1; echo "k=$k rc=$?"
tail -1 gpurun_out/bench_k$k.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d['timeline']
print('value',d['value'],'ms',d['ms_per_step'],'miss/tok',d['miss_loads_per_token'],'hit',d['hit_rate'])
print({k:v['avg_us'] for k,v in t['kernels'].items()}, t['token_span_us'])"
done
MOE_COPY_TRACE=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 8 > gpurun_out/bench_trace.log 2> gpurun_out/copy_trace.log; echo "trace rc=$?"
grep -c "demand chunk" gpurun_out/copy_trace.log
