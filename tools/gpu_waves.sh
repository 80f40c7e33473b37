#!/bin/bash
# A/B of resident waves per GEMV launch (MOE_MG_WAVES="qkv,wo,up,down"):
# bench lines (no e2e / prompts / CPU leg) for each setting, base first and last.
mkdir -p gpurun_out
for w in ${WAVES:-1,1,1,1 1,1,2,2 1,1,2,1 2,2,1,1 1,1,1,1}; do
  MOE_MG_WAVES=$w timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-prompts ${BENCH_ARGS:-} \
    > gpurun_out/waves_$w.json 2> gpurun_out/waves_$w.err
  echo "waves $w rc=$?"
  grep '^{' gpurun_out/waves_$w.json | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d.get('timeline',{}).get('kernels',{})
print('$w', d['value'], d['roofline']['avg_launch_us'], {k: t[k]['median_us'] for k in ('qkv','wo','tail','expert_up','expert_down') if k in t})"
done
