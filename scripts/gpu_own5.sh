mkdir -p gpurun_out/own5
O=gpurun_out/own5
for cfg in "1 1" "1 0" "2 1" "0 1" "3 1"; do
  set -- $cfg
  PN_FLOW_HOLD=$1 PN_FLOW_PICK=$2 PN_MGS_TRACE=$O/trace_$1_$2.txt timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('hold $1 pick $2', round(d['ms_per_step'],2), round(d['roofline']['seconds']*1e3,2))"
done
for t in 100 120 170; do
  PN_MGS_TAIL=$t timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('tail $t', round(d['ms_per_step'],2), round(d['roofline']['seconds']*1e3,2))"
done
