#!/bin/bash
# MGS changes: parity suites, then the three levels' step timing and an ncu
# capture of the cdd pipe kernel.
cd "$(dirname "$0")/.."
T=${TAG:-r02i}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_fullsize.py tests/test_mgs_small.py tests/test_flow_sched.py tests/test_config_parity.py tests/test_batch.py -q -p no:cacheprovider -x > gpurun_out/${T}_mgs_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_mgs_tests.log
for base in d dd qd; do
  timeout 300 python bench.py --base $base --no-extras --no-cpu-baseline --steps 10 > gpurun_out/${T}_mgs_$base.json 2>&1
done
OUT=gpurun_out/${T}_ncu_pipe_dd timeout 600 bash scripts/ncu_kernel.sh k_mgs_pipe --base dd
tail -3 gpurun_out/${T}_mgs_tests.log
