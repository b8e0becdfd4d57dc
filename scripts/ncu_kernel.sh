#!/bin/bash
# ncu --set full capture of one kernel launch (regex $1) during a short bench run ($2...)
cd "$(dirname "$0")/.."
K=$1; shift; OUT=${OUT:-gpurun_out/ncu_$K}
ncu --set full --clock-control none --import-source on -k "regex:$K" -c ${COUNT:-1} -o $OUT -f python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 1 "$@" > ${OUT}.log 2>&1
echo "ncu_rc=$?" >> ${OUT}.log
tail -2 ${OUT}.log
