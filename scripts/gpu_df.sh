mkdir -p gpurun_out/df
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/df
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_batch.py -m gpu -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -2
for b in dd d; do timeout 600 python bench.py --base $b --steps 5 --warmup 2 --no-cpu-baseline > $O/b$b.json 2>$O/b.err; tail -2 $O/b.err
python -c "import json;d=json.load(open('$O/b$b.json'));print('c$b ms/step %.2f'%d['ms_per_step'],{k:round(v,2) for k,v in d['phases_ms'].items()}, 'factor', round(d['roofline']['seconds']*1e3,2), 'bsub', round(d['backsub']['seconds']*1e3,2))"; done
