# flow kernel q handling in the update: 0 reload via L2, 1 registers, 2 L1 prefetch
set -x
mkdir -p gpurun_out/qm
O=gpurun_out/qm
for qm in 1 2; do PN_FLOW_QM=$qm timeout 900 python -m pytest tests/test_fullsize.py tests/test_flow_sched.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "headline or tail or flow" 2>&1 | tail -2; done
for qm in 0 1 2 0 1 2; do
  PN_FLOW_QM=$qm timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('qm $qm', d['ms_per_step'], d['roofline']['seconds'])"
done
