# flow kernel column ownership (rr vs snake) x hold
set -x
mkdir -p gpurun_out/own
O=gpurun_out/own
PN_FLOW_OWN=snake PN_FLOW_HOLD=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "mgs or least or tail or headline or step" 2>&1 | tail -3
for cfg in "rr 0" "snake 0" "snake 1" "snake 2" "rr 1"; do
  set -- $cfg
  PN_FLOW_OWN=$1 PN_FLOW_HOLD=$2 PN_MGS_TRACE=$O/trace_$1_$2.txt timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('own $1 hold $2', d['ms_per_step'], d['roofline']['seconds'])"
done
for f in sim/*.txt; do [ -f $f ] || continue
  PN_FLOW_OWN=$f PN_FLOW_HOLD=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('own $f hold 1', d['ms_per_step'], d['roofline']['seconds'])"
done
