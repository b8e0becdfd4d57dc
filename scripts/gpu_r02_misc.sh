#!/bin/bash
# CLI + C-ABI collective tests, and a pivot-time trace of the cqd MGS.
cd "$(dirname "$0")/.."
T=${TAG:-r02k}
timeout 900 python -m pytest tests/test_cli.py tests/test_batch.py -q -p no:cacheprovider > gpurun_out/${T}_misc_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_misc_tests.log
PN_MGS_TRACE=gpurun_out/${T}_trace_qd.txt timeout 300 python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 1 --e2e-steps 1 > gpurun_out/${T}_trace_bench.json 2>&1
tail -3 gpurun_out/${T}_misc_tests.log
