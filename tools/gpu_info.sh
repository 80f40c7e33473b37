#!/bin/bash
# Box facts the bench and the CPU reference arm depend on (cores, RAM, NUMA, PCIe).
mkdir -p gpurun_out
{ nproc; free -g; lscpu | head -20; nvidia-smi; nvidia-smi topo -m; numactl -H 2>/dev/null; } > gpurun_out/box.txt 2>&1
