#!/bin/bash
# Profiling round trip: ncu launch list of the C2 bench, one ncu --set full
# capture of one layer's kernels (QKV, attention, Wo, tail, W1||W3, W2), and
# compute-sanitizer (memcheck, racecheck, synccheck) on the smoke.
#   gpurun --timeout 3000 -- 'bash tools/gpu_profile.sh [launch] [full] [san]'
set -u
what=" ${*:-launch full san} "
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
SAN=/usr/local/cuda/bin/compute-sanitizer
if [[ $what == *" launch "* ]]; then
  MOE_NCU_RANGE=1 timeout 900 $NCU --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
     --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-prompts ${BENCH_ARGS:-} > gpurun_out/ncu_launch.log 2>&1
  echo "ncu launches rc=$?"
fi
if [[ $what == *" full "* ]]; then
  MOE_NCU_RANGE=1 timeout 1200 $NCU --profile-from-start off --set full --clock-control none --import-source on \
     -k "regex:${NCU_KERNEL:-k_mgemv|k_tail|k_attention}" -s ${NCU_SKIP:-6} -c ${NCU_COUNT:-6} -o gpurun_out/prof -f \
     python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-prompts ${BENCH_ARGS:-} > gpurun_out/ncu_full.log 2>&1
  echo "ncu full rc=$?"
fi
if [[ $what == *" san "* ]]; then
  for tool in memcheck racecheck synccheck; do
    timeout 900 $SAN --tool $tool --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" \
      > gpurun_out/sanitizer_$tool.log 2>&1
    echo "sanitizer $tool rc=$?" | tee -a gpurun_out/sanitizer_$tool.log
  done
fi
