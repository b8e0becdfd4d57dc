#!/bin/bash
# k_mgs_pipe block ownership: MGS parity, then cd / cdd timing per (QB, bw).
cd "$(dirname "$0")/.."
T=${TAG:-r02h}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize.py tests/test_mgs_small.py tests/test_flow_sched.py -q -p no:cacheprovider -x > gpurun_out/${T}_pipe_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_pipe_tests.log
for bw in 1 2 4 8; do
  PN_PIPE_BW=$bw timeout 300 python bench.py --base d --no-extras --no-cpu-baseline --steps 10 > gpurun_out/${T}_pipe_d_bw$bw.json 2>&1
done
for cfg in "1 1" "2 2" "2 4" "1 2"; do set -- $cfg
  PN_PIPE_QB=$1 PN_PIPE_BW=$2 timeout 300 python bench.py --base dd --no-extras --no-cpu-baseline --steps 10 > gpurun_out/${T}_pipe_dd_qb$1_bw$2.json 2>&1
done
tail -3 gpurun_out/${T}_pipe_tests.log
