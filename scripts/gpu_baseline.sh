# re-entry check: parity tests, smoke, default bench, launch list and full
# ncu captures (with dram bytes) of the dominant kernels of the default bench
mkdir -p gpurun_out/base
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/base
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x 2>&1 | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_default.json 2> $O/bench_default.err; tail -2 $O/bench_default.err; cat $O/bench_default.json
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_cqd.csv $B > /dev/null 2>$O/launch.err
for spec in "mgs:k_mgs_flow" "tree:k_mono_tree" "seg:k_segments"; do
  name=${spec%%:*}; kern=${spec#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kern -c 1 -o /tmp/prof_$name $B > /dev/null 2>$O/$name.err
  ncu -i /tmp/prof_$name.ncu-rep --page details --csv > $O/${name}_details.csv 2>>$O/$name.err
  ncu -i /tmp/prof_$name.ncu-rep --page raw --csv > $O/${name}_raw.csv 2>>$O/$name.err
  ncu -i /tmp/prof_$name.ncu-rep --page source --csv 2>>$O/$name.err | gzip > $O/${name}_source.csv.gz
done
du -sh gpurun_out
