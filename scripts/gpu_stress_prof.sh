#!/bin/bash
cd "$(dirname "$0")/.."
export PATH=/usr/local/cuda/bin:$PATH
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_stress.csv python bench.py --family stress --steps 1 --warmup 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mono_warp -c 1 -o gpurun_out/ncu_stress_warp python bench.py --family stress --steps 1 --warmup 0 > /dev/null 2>&1
