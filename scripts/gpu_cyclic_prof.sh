#!/bin/bash
# per-kernel launch times of the cyclic n-roots evaluation (the paper's Table)
cd "$(dirname "$0")/.."
export PATH=/usr/local/cuda/bin:$PATH
T=${TAG:-r02n}
for spec in "d 512" "qd 448"; do set -- $spec
  timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${T}_cyc_$1.csv python bench.py --family cyclic --base $1 --dim $2 --steps 1 --warmup 1 > /dev/null 2>gpurun_out/${T}_cyc_$1.err
done
