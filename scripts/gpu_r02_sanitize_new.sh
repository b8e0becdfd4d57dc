#!/bin/bash
# compute-sanitizer over the kernels added late in round 2: tall flow
# variants (512-thread real qd / complex dd, 8-row complex dd up to 2048
# rows) and the pipe kernel's cluster (PAIR) variant.
cd "$(dirname "$0")/.."
export PATH=/usr/local/cuda/bin:$PATH
T=${TAG:-r02n}
S="compute-sanitizer --print-limit 20 --error-exitcode 99"
K1='tall and (cdd-4096-48 or rqd-2100-90 or cdd-1600-120)'
K2='least_squares_vs_oracle and pipe/pair and ((cd-256-256) or (rd-512-512))'
for tool in memcheck synccheck; do
  X=""; [ $tool = synccheck ] && X="--num-cuda-barriers 64"
  $S --tool $tool $X python -m pytest tests/test_config_parity.py -q -p no:cacheprovider -x -k "$K1" > gpurun_out/${T}_${tool}_tall.log 2>&1
  echo "rc=$?" >> gpurun_out/${T}_${tool}_tall.log
  $S --tool $tool $X python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "$K2" > gpurun_out/${T}_${tool}_pair.log 2>&1
  echo "rc=$?" >> gpurun_out/${T}_${tool}_pair.log
done
$S --tool racecheck python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "least_squares_vs_oracle and pipe/pair and cd-256-256" > gpurun_out/${T}_racecheck_pair.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_racecheck_pair.log
for f in gpurun_out/${T}_*.log; do echo "$f: $(grep -E 'passed|failed|ERROR SUMMARY|RACECHECK SUMMARY' $f | tr '\n' ' ') $(tail -1 $f)"; done
