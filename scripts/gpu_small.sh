# one-CTA MGS for m <= 32
set -x
mkdir -p gpurun_out/small
O=gpurun_out/small
timeout 1500 python -m pytest tests/test_mgs_small.py tests/test_gpu_parity.py tests/test_step_graph.py tests/test_acceptance_gpu.py -m gpu -q -x --timeout 900 -p no:cacheprovider -k "small or golden or graph or criterion or c1 or newton" 2>&1 | tail -3
for b in d dd qd; do for g in small dataflow; do
  PN_MGS_MODE=$g timeout 600 python bench.py --dim 32 --terms 32 --k 8 --base $b --steps 50 --warmup 10 --no-cpu-baseline > $O/m.json 2>$O/m.err
  python -c "import json; d=json.loads(open('$O/m.json').read().strip().splitlines()[-1]); print('$b $g', round(d['ms_per_step'],4), d['e2e']['value'], d['phases_ms'])"
done; done
