#!/bin/bash
# A/B timing: run bench.py --base $BASE under each environment setting given as arguments ("VAR=val ...").
cd "$(dirname "$0")/.."
T=${TAG:-ab}
i=0
for cfg in "$@"; do
  for rep in 1 2; do
    env $cfg timeout 300 python bench.py --base ${BASE:-dd} --no-extras --no-cpu-baseline --steps 10 > gpurun_out/${T}_${i}_${rep}.json 2>&1
  done
  echo "$i $cfg" >> gpurun_out/${T}_index.txt
  i=$((i+1))
done
