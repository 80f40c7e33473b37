#!/bin/bash
# round-end style check: smoke, GPU tests, C2 (+CPU baseline) and C3 bench,
# reference arm, ncu launch list of the C2 decode, ncu full of the W1/W3 and W2 GEMVs
mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=${MOE_WAIT_TIMEOUT_MS:-20000}
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c2.log 2>&1; echo "bench c2 rc=$?"
timeout 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo "bench c3 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
MOE_SERIAL_COPIES=1 MOE_NCU_RANGE=1 timeout 900 /usr/local/cuda/bin/ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
   --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:k_gemv -s 5 -c 1 -o gpurun_out/gemv3_up -f python tools/gemv_one.py 3 4096 14336 4 8 > gpurun_out/ncu_up.log 2>&1; echo "ncu up rc=$?"
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:k_gemv -s 5 -c 1 -o gpurun_out/gemv3_down -f python tools/gemv_one.py 3 14336 4096 2 8 > gpurun_out/ncu_down.log 2>&1; echo "ncu down rc=$?"
