#!/bin/bash
# tests + C2 and C3 bench + ncu launch list (round-trip helper)
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=${MOE_WAIT_TIMEOUT_MS:-20000}
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
MOE_FAULTHANDLER=500 timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; echo "bench c2 rc=$?"
MOE_FAULTHANDLER=500 timeout 600 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo "bench c3 rc=$?"
MOE_SERIAL_COPIES=1 MOE_NCU_RANGE=1 timeout 900 /usr/local/cuda/bin/ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
   --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu rc=$?"
