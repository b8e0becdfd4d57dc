# build-free GPU iteration: parity tests, benches, optional ncu captures
mkdir -p gpurun_out/iter
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -25
for b in qd dd d; do timeout 600 python bench.py --base $b --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/iter/bench_c$b.json 2>gpurun_out/iter/bench_c$b.err; tail -3 gpurun_out/iter/bench_c$b.err; done
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1"
for spec in $PROF; do
  name=${spec%%:*}; kern=${spec#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kern -c 1 -o /tmp/prof_$name $B > /dev/null 2>gpurun_out/iter/$name.err
  ncu -i /tmp/prof_$name.ncu-rep --page details --csv > gpurun_out/iter/${name}_details.csv 2>>gpurun_out/iter/$name.err
  ncu -i /tmp/prof_$name.ncu-rep --page raw --csv > gpurun_out/iter/${name}_raw.csv 2>>gpurun_out/iter/$name.err
  ncu -i /tmp/prof_$name.ncu-rep --page source --csv 2>>gpurun_out/iter/$name.err | gzip > gpurun_out/iter/${name}_source.csv.gz
done
du -sh gpurun_out
