mkdir -p gpurun_out/prof
export PATH=/usr/local/cuda/bin:$PATH
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_cqd.csv $B > /dev/null 2>gpurun_out/prof/launch.err
for spec in "mgs:k_mgs_sweep:-s 40" "tree:k_mono_tree:" "seg:k_segments:"; do
  name=${spec%%:*}; rest=${spec#*:}; kern=${rest%%:*}; extra=${rest#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kern $extra -c 1 -o /tmp/prof_$name $B > /dev/null 2>gpurun_out/prof/$name.err
  ncu -i /tmp/prof_$name.ncu-rep --page details --csv > gpurun_out/prof/${name}_details.csv 2>>gpurun_out/prof/$name.err
  ncu -i /tmp/prof_$name.ncu-rep --page raw --csv > gpurun_out/prof/${name}_raw.csv 2>>gpurun_out/prof/$name.err
  ncu -i /tmp/prof_$name.ncu-rep --page source --csv > gpurun_out/prof/${name}_source.csv 2>>gpurun_out/prof/$name.err
done
for b in d dd; do timeout 600 python bench.py --base $b --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/prof/bench_c$b.json 2>gpurun_out/prof/bench_c$b.err; done
gzip -f gpurun_out/prof/*_source.csv
du -sh gpurun_out; ls -la gpurun_out/prof
