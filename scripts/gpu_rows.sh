#!/bin/bash
# Row evaluation: parity suite, eval timing against K1+K2, ncu of k_eval_rows (cd).
cd "$(dirname "$0")/.."
T=${TAG:-r02c}
timeout 900 python -m pytest tests/test_eval_rows.py tests/test_fullsize.py tests/test_batch.py -q -p no:cacheprovider -x > gpurun_out/${T}_rows_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_rows_tests.log
for base in d dd qd; do
  for r in 0 1; do
    PN_EVAL_ROWS=$r timeout 300 python bench.py --base $base --no-extras --no-cpu-baseline --steps 10 > gpurun_out/${T}_rows_${base}_${r}.json 2>&1
  done
done
PN_EVAL_ROWS=1 OUT=gpurun_out/${T}_ncu_rows_cd timeout 600 bash scripts/ncu_kernel.sh k_eval_rows --base d
tail -3 gpurun_out/${T}_rows_tests.log
