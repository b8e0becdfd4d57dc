mkdir -p gpurun_out/pipe
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/pipe
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_fullsize.py -m gpu -q --timeout 600 -p no:cacheprovider -x -k "least_squares or breakdown or newton or c3" 2>&1 | tail -3
for b in dd d; do for mode in pipe dataflow; do PN_MGS_MODE=$mode timeout 600 python bench.py --base $b --steps 5 --warmup 2 --no-cpu-baseline > $O/b.json 2>$O/b.err; tail -2 $O/b.err
python -c "import json;d=json.load(open('$O/b.json'));print('c$b $mode ms/step %.2f'%d['ms_per_step'],{k:round(v,2) for k,v in d['phases_ms'].items()}, 'factor', round(d['roofline']['seconds']*1e3,2))"; done; done
