# flow kernel 128 x 8 (3 CTAs/SM) vs 256 x 4; schedule tests
set -x
mkdir -p gpurun_out/nt
O=gpurun_out/nt
timeout 900 python -m pytest tests/test_flow_sched.py -m gpu -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -3
PN_FLOW_NT=128 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "mgs or least or tail or headline" 2>&1 | tail -3
for cfg in "256 1" "128 1" "128 0" "128 2"; do
  set -- $cfg
  PN_FLOW_NT=$1 PN_FLOW_HOLD=$2 PN_MGS_TRACE=$O/trace_$1_$2.txt timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('nt $1 hold $2', d['ms_per_step'], d['roofline']['seconds'])"
done
