mkdir -p gpurun_out/fc
O=gpurun_out/fc
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $O/t.log 2>&1; tail -3 $O/t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for i in 1 2; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('cqd', round(d['ms_per_step'],2), round(d['roofline']['seconds']*1e3,2), d['phases_ms'])"
done
timeout 900 python bench.py --converge --rows 1536 --max-iters 10 > $O/c4o.json 2>$O/c4o.err; tail -1 $O/c4o.json | cut -c1-300
