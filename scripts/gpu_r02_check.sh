#!/bin/bash
# Round-2 check: GPU suite, sanitizers on the changed kernels, default bench.
cd "$(dirname "$0")/.."
T=${TAG:-r02j}
export PATH=/usr/local/cuda/bin:$PATH
python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/${T}_tests.log 2>&1
echo "tests_rc=$?" >> gpurun_out/${T}_tests.log
S="compute-sanitizer --print-limit 20 --error-exitcode 99"
$S --tool racecheck python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "back_substitution and (look or blocked) and (77 or 300 or 33 or 64)" > gpurun_out/${T}_racecheck_bsub.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_racecheck_bsub.log
$S --tool memcheck python -m pytest tests/test_eval_rows.py -q -p no:cacheprovider -x -k "not full_size" > gpurun_out/${T}_memcheck_rows.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_memcheck_rows.log
$S --tool racecheck python -m pytest tests/test_eval_rows.py -q -p no:cacheprovider -x -k "every_tree_base or ragged" > gpurun_out/${T}_racecheck_rows.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_racecheck_rows.log
$S --tool synccheck --num-cuda-barriers 64 python -m pytest tests/test_eval_rows.py -q -p no:cacheprovider -x -k "every_tree_base" > gpurun_out/${T}_synccheck_rows.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_synccheck_rows.log
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
tail -2 gpurun_out/${T}_tests.log
