#!/bin/bash
# EP bench path end to end with 2 ranks sharing GPU 0 (timings meaningless; checks the plumbing)
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=60000 MOE_BENCH_DEVICE=0
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ep2.log 2>&1; echo "ep2 rc=$?"
tail -1 gpurun_out/bench_ep2.log | cut -c1-400
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --impl reference --gpus 2 --steps 1 --warmup 3 > gpurun_out/bench_ep2_ref.log 2>&1; echo "ep2 ref rc=$?"
tail -1 gpurun_out/bench_ep2_ref.log | cut -c1-200
