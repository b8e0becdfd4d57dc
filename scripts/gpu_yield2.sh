mkdir -p gpurun_out/yield2
O=gpurun_out/yield2
for cfg in "0 1" "20000 1" "50000 1" "20000 2" "100000 1" "50000 2"; do
  set -- $cfg
  PN_FLOW_YIELD=$1 PN_FLOW_YIELD_F=$2 PN_MGS_TRACE=$O/trace_$1_$2.txt timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('yield $1 f $2', round(d['ms_per_step'],2), round(d['roofline']['seconds']*1e3,2))"
done
