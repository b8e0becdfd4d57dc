mkdir -p gpurun_out/smmap
O=gpurun_out/smmap
timeout 900 python -m pytest tests/test_flow_sched.py tests/test_fullsize.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "flow or headline or tail" > $O/t.log 2>&1; tail -1 $O/t.log
for v in 1 0 1 0; do
  PN_FLOW_SMMAP=$v PN_MGS_TRACE=$O/trace_$v.txt timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('smmap $v', round(d['ms_per_step'],2), round(d['roofline']['seconds']*1e3,2))"
done
