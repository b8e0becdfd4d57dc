# cdd/cd: flow kernel (with hold) vs pipe
set -x
mkdir -p gpurun_out/ddflow
O=gpurun_out/ddflow
for b in dd d; do for cfg in "pipe 1" "flow 0" "flow 1" "flow 2"; do
  set -- $cfg
  PN_MGS_MODE=$1 PN_FLOW_HOLD=$2 timeout 600 python bench.py --base $b --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('$b $1 hold $2', d['ms_per_step'], d['roofline']['seconds'])"
done; done
