#!/bin/bash
# Newton-step size sweep: F(dim, dim, 32) for dim = 256..1024 on every complex level
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/sweep
for b in d dd qd; do
  for dim in 256 512 768 1024; do
    timeout 600 python bench.py --base $b --dim $dim --terms $dim --no-extras --no-cpu-baseline --steps 5 --warmup 3 \
      > gpurun_out/sweep/step_${b}_${dim}.json 2> gpurun_out/sweep/step_${b}_${dim}.err
  done
done
ls gpurun_out/sweep | wc -l
