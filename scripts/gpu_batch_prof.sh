# batched C5 path: launch list + full capture of the solve kernel and the tree kernel
mkdir -p gpurun_out/bprof
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/bprof
B="python bench.py --batch ${NB:-296} --dim 256 --terms 256 --base dd --steps 1 --warmup 1 --max-iters 2"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file $O/launches.csv $B > /dev/null 2>$O/launch.err
for spec in ${PROF:-"solve:k_solve_batch" "tree:k_mono_tree" "seg:k_segments"}; do
  name=${spec%%:*}; kern=${spec#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kern -s 1 -c 1 -o /tmp/prof_$name $B > /dev/null 2>$O/$name.err
  ncu -i /tmp/prof_$name.ncu-rep --page details --csv > $O/${name}_details.csv 2>>$O/$name.err
  ncu -i /tmp/prof_$name.ncu-rep --page raw --csv > $O/${name}_raw.csv 2>>$O/$name.err
  ncu -i /tmp/prof_$name.ncu-rep --page source --csv 2>>$O/$name.err | gzip > $O/${name}_source.csv.gz
done
ls -la $O
