# compare library variants on the cqd (and optionally other) benches
mkdir -p gpurun_out/var
export PATH=/usr/local/cuda/bin:$PATH
if [ -n "$TESTS" ]; then timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -5; fi
for v in $VARIANTS; do
  name=${v%%=*}; lib=${v#*=}
  for b in $LEVELS; do
    PN_LIB=$lib timeout 600 python bench.py --base $b --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/var/${name}_c$b.json 2>gpurun_out/var/${name}_c$b.err
    python -c "import json;d=json.load(open('gpurun_out/var/${name}_c$b.json'));print('$name','c$b','ms/step %.2f'%d['ms_per_step'],{k:round(v,2) for k,v in d['phases_ms'].items()})" 2>&1 | tail -1
  done
done
for spec in $PROF; do
  name=${spec%%:*}; rest=${spec#*:}; kern=${rest%%:*}; lib=${rest#*:}
  PN_LIB=$lib timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kern -c 1 -o /tmp/prof_$name python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>gpurun_out/var/$name.err
  ncu -i /tmp/prof_$name.ncu-rep --page details --csv > gpurun_out/var/${name}_details.csv 2>>gpurun_out/var/$name.err
  ncu -i /tmp/prof_$name.ncu-rep --page raw --csv > gpurun_out/var/${name}_raw.csv 2>>gpurun_out/var/$name.err
  ncu -i /tmp/prof_$name.ncu-rep --page source --csv 2>>gpurun_out/var/$name.err | gzip > gpurun_out/var/${name}_source.csv.gz
done
