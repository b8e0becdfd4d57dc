# batched C5: full captures of the big batched tree/segments/solve launches
mkdir -p gpurun_out/bprof2
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/bprof2
B="python bench.py --batch 296 --dim 256 --terms 256 --base dd --steps 1 --warmup 1 --max-iters 1"
for spec in "tree:k_mono_tree" "seg:k_segments" "solve:k_solve_batch"; do
  name=${spec%%:*}; kern=${spec#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kern -s 2 -c 1 -o /tmp/prof_$name $B > /dev/null 2>$O/$name.err
  ncu -i /tmp/prof_$name.ncu-rep --page details --csv > $O/${name}_details.csv 2>>$O/$name.err
  ncu -i /tmp/prof_$name.ncu-rep --page raw --csv > $O/${name}_raw.csv 2>>$O/$name.err
  ncu -i /tmp/prof_$name.ncu-rep --page source --csv 2>>$O/$name.err | gzip > $O/${name}_source.csv.gz
done
python scripts/ncu_summary.py $O/tree_raw.csv $O/seg_raw.csv $O/solve_raw.csv
