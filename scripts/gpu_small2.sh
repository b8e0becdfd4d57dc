set -x
mkdir -p gpurun_out/small
O=gpurun_out/small
timeout 900 python -m pytest tests/test_mgs_small.py tests/test_step_graph.py -m gpu -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -2
for b in d; do for i in 1 2; do
  timeout 600 python bench.py --dim 32 --terms 32 --k 8 --base $b --steps 50 --warmup 10 > $O/m.json 2>$O/m.err
  python -c "import json; d=json.loads(open('$O/m.json').read().strip().splitlines()[-1]); print('$b', round(d['ms_per_step'],4), round(d['e2e']['value']), d['phases_ms'], d['roofline']['seconds'], d['cpu_baseline'])"
done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_c1.csv python bench.py --dim 32 --terms 32 --k 8 --base d --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>$O/n.err
python scripts/ncu_summary.py $O/launch_c1.csv
