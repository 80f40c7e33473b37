#!/bin/bash
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=20000
for dir in _wt .; do
(cd $dir && timeout 600 python bench.py --no-cpu-baseline --no-e2e > /tmp/b.log 2>&1; echo "$dir rc=$?"; tail -1 /tmp/b.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d['timeline']
print('value',d['value'],'ms',d['ms_per_step'])
print({k:v.get('median_us',v['avg_us']) for k,v in t['kernels'].items()}); p=t['phases_us']; print({k:p[k] for k in ('attention','tail')})")
done
