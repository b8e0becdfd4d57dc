# graph-replayed Newton step for small systems
set -x
mkdir -p gpurun_out/graph
O=gpurun_out/graph
timeout 900 python -m pytest tests/test_step_graph.py tests/test_acceptance_gpu.py tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "graph or criterion or newton or c1" 2>&1 | tail -3
for b in d dd qd; do for g in 1 0; do
  PN_GRAPH=$g timeout 600 python bench.py --dim 32 --terms 32 --k 8 --base $b --steps 50 --warmup 10 --no-cpu-baseline > $O/m.json 2>$O/m.err
  python -c "import json; d=json.loads(open('$O/m.json').read().strip().splitlines()[-1]); print('$b graph $g', round(d['ms_per_step'],4), d['e2e']['value'], d['gpu_launches'], d['phases_ms'])"
done; done
tail -3 $O/m.err
