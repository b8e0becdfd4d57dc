# flow kernel hold rule with a lag bound
set -x
mkdir -p gpurun_out/hold2
O=gpurun_out/hold2
for cfg in "1 1073741824" "1 4" "1 16" "1 64" "2 16" "2 64" "1 256"; do
  set -- $cfg
  PN_FLOW_HOLD=$1 PN_FLOW_LAG=$2 PN_MGS_TRACE=$O/trace_$1_$2.txt timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('hold $1 lag $2', d['ms_per_step'], d['roofline']['seconds'])"
done
