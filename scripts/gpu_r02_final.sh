#!/bin/bash
# Round-2 final pass: GPU suite, smoke, default bench line, reference arm,
# cyclic families (the large-k warp kernel changed late in the round).
cd "$(dirname "$0")/.."
T=${TAG:-r02z}
python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/${T}_tests.log 2>&1
echo "tests_rc=$?" >> gpurun_out/${T}_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python bench.py --family cyclic --base d --steps 5 > gpurun_out/${T}_cyc_d.json 2>&1
python bench.py --family cyclic --base dd --steps 3 > gpurun_out/${T}_cyc_dd.json 2>&1
python bench.py --family cyclic --base qd --steps 2 --warmup 3 > gpurun_out/${T}_cyc_qd.json 2>&1
tail -3 gpurun_out/${T}_tests.log
