# flow kernel: hold lagging work on the CTA next on the critical path
set -x
mkdir -p gpurun_out/hold
O=gpurun_out/hold
PN_FLOW_HOLD=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize.py tests/test_tree_pad.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "mgs or least or tail or headline or step or pad" 2>&1 | tail -3
for h in 0 1 2 3 0 1; do
  PN_FLOW_HOLD=$h PN_MGS_TRACE=$O/trace_$h.txt timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/b_$h.json 2>$O/b_$h.err
  python -c "import json; d=json.loads(open('$O/b_$h.json').read().strip().splitlines()[-1]); print('hold $h', d['ms_per_step'], d['roofline']['seconds'])"
done
