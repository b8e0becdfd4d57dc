mkdir -p gpurun_out/sleep
O=gpurun_out/sleep
for v in 100 20 0 400 100 20; do
  PN_FLOW_SLEEP=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('sleep $v', round(d['ms_per_step'],2), round(d['roofline']['seconds']*1e3,2))"
done
