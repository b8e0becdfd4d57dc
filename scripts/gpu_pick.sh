# flow kernel lagging-column pick rule
set -x
mkdir -p gpurun_out/pick
O=gpurun_out/pick
PN_FLOW_PICK=1 timeout 900 python -m pytest tests/test_fullsize.py tests/test_flow_sched.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "headline or tail or flow" 2>&1 | tail -2
for cfg in "0 1" "1 1" "1 0" "1 2"; do
  set -- $cfg
  PN_FLOW_PICK=$1 PN_FLOW_HOLD=$2 PN_MGS_TRACE=$O/trace_$1_$2.txt timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('pick $1 hold $2', d['ms_per_step'], d['roofline']['seconds'])"
done
