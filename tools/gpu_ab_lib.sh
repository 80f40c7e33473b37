#!/bin/bash
# A/B of the product library against one variant (tools/ab_build.sh TAG ...):
# GPU tests of the product library, then C2 bench lines alternating the two.
#   gpurun -- 'AB_TAG=nocl bash tools/gpu_ab_lib.sh'
mkdir -p gpurun_out
tag=${AB_TAG:?set AB_TAG}
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do
  for v in base $tag; do
    if [ $v = base ]; then unset MOE_LIB_PATH; else export MOE_LIB_PATH=$PWD/paper_2312_17238_b200/libmoeb200_ab_$tag.so; fi
    timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-prompts --no-secondary > gpurun_out/ab_${v}_$i.json 2> gpurun_out/ab_${v}_$i.err
    grep '^{' gpurun_out/ab_${v}_$i.json | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d.get('timeline',{}).get('kernels',{})
print('$v', d['value'], {k: (t[k]['median_us'], t[k].get('phase_marks_us',{}).get('0')) for k in ('qkv','wo','tail','expert_up','expert_down') if k in t})"
  done
done
unset MOE_LIB_PATH
