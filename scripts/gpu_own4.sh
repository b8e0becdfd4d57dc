mkdir -p gpurun_out/own4
O=gpurun_out/own4
for t in smsnake_alt smsnake_abba smsnake_ph1 smsnake_ba smsnake_par smsnake_alt; do
  PN_FLOW_OWN=scripts/own/$t.txt PN_MGS_TRACE=$O/trace_$t.txt timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('$t', round(d['ms_per_step'],2), round(d['roofline']['seconds']*1e3,2))"
done
