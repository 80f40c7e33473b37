mkdir -p gpurun_out
export MOE_WAIT_TIMEOUT_MS=15000
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 300 python tools/gemv_bench.py > gpurun_out/gemv_bench.log 2>&1; echo "gemv rc=$?"
MOE_COPY_CHUNK_MB=1000 timeout 300 python tools/debug_mixtral.py 2 2 2 > gpurun_out/dbg_c3_nochunk.log 2>&1; echo "nochunk rc=$?"
MOE_GRAPH=0 timeout 300 python tools/debug_mixtral.py 2 2 2 > gpurun_out/dbg_c3_nograph.log 2>&1; echo "nograph rc=$?"
MOE_PDL=0 timeout 300 python tools/debug_mixtral.py 2 2 2 > gpurun_out/dbg_c3_nopdl.log 2>&1; echo "nopdl rc=$?"
MOE_DEBUG=1 timeout 300 python tools/debug_mixtral.py 2 2 2 > gpurun_out/dbg_c3_debug.log 2>&1; echo "debug rc=$?"
