#!/bin/bash
# Round-2 GPU pass: full GPU suite, default bench line, paper families.
cd "$(dirname "$0")/.."
T=${TAG:-r02b}
python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/${T}_tests.log 2>&1
echo "tests_rc=$?" >> gpurun_out/${T}_tests.log
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python bench.py --family cyclic --base d --steps 5 > gpurun_out/${T}_cyc_d.json 2>&1
python bench.py --family cyclic --base dd --steps 3 > gpurun_out/${T}_cyc_dd.json 2>&1
python bench.py --family cyclic --base qd --steps 2 --warmup 1 > gpurun_out/${T}_cyc_qd.json 2>&1
python bench.py --family chandra --base dd > gpurun_out/${T}_chandra_dd.json 2>&1
python bench.py --family chandra --base qd > gpurun_out/${T}_chandra_qd.json 2>&1
tail -3 gpurun_out/${T}_tests.log
