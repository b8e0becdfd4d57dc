#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck over the pipe MGS kernel
# (both prefetch points) on small parity cases.
cd "$(dirname "$0")/.."
export PATH=/usr/local/cuda/bin:$PATH
T=${TAG:-r02s}
S="compute-sanitizer --print-limit 20 --error-exitcode 99"
K='least_squares_vs_oracle and pipe and ((cd-256-256) or (rdd-512-200) or (cdd-256-100))'
for tool in racecheck synccheck memcheck; do
  X=""; [ $tool = synccheck ] && X="--num-cuda-barriers 64"
  $S --tool $tool $X python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "$K" > gpurun_out/${T}_${tool}_pipe.log 2>&1
  echo "rc=$?" >> gpurun_out/${T}_${tool}_pipe.log
done
tail -3 gpurun_out/${T}_*_pipe.log
