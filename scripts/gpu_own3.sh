mkdir -p gpurun_out/own3
O=gpurun_out/own3
for t in rr smsnake_alt smsnake_lpt smrr_lpt smsnake_lpt smsnake_alt; do
  PN_FLOW_OWN=scripts/own/$t.txt PN_MGS_TRACE=$O/trace_$t.txt timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('$t', round(d['ms_per_step'],2), round(d['roofline']['seconds']*1e3,2))"
done
PN_FLOW_OWN=scripts/own/smsnake_lpt.txt timeout 900 python -m pytest tests/test_fullsize.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "headline" > $O/t.log 2>&1; tail -1 $O/t.log
