mkdir -p gpurun_out/flow2
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/flow2
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cqd.json 2>$O/bench_cqd.err; tail -3 $O/bench_cqd.err
python -c "import json;d=json.load(open('$O/bench_cqd.json'));print('cqd ms/step %.2f'%d['ms_per_step'],{k:round(v,2) for k,v in d['phases_ms'].items()})"
timeout 900 python bench.py --converge --rows 1536 --max-iters 10 > $O/c4_over.json 2>$O/c4_over.err; python -c "import json;d=json.load(open('$O/c4_over.json'));print('c4 over ms/step %.2f'%d['ms_per_step'], d['iterations'], d['f_norm'][-1])"
