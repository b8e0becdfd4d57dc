# hold=1 x tail size / variant
set -x
mkdir -p gpurun_out/own2
O=gpurun_out/own2
for cfg in "a 0" "b 0" "a 100" "b 200" "c 0" "a 120"; do
  set -- $cfg
  T=$2; [ "$T" = "0" ] && T=""
  PN_FLOW_OWN=rr PN_FLOW_HOLD=1 PN_MGS_TAIL_VARIANT=$1 PN_MGS_TAIL=$T PN_MGS_TRACE=$O/trace_$1_$2.txt timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('variant $1 tail $2', d['ms_per_step'], d['roofline']['seconds'])"
done
