mkdir -p gpurun_out/own6
O=gpurun_out/own6
for t in sm_r6s1 sm_r6rev sm_r6rev_s1 smsnake_alt sm_r6s1; do
  PN_FLOW_OWN=scripts/own/$t.txt PN_FLOW_SMMAP=0 PN_MGS_TRACE=$O/trace_$t.txt timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('$t', round(d['ms_per_step'],2), round(d['roofline']['seconds']*1e3,2))"
done
