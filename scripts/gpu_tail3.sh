mkdir -p gpurun_out/tail
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/tail
for V in a b; do PN_MGS_TAIL_VARIANT=$V timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > $O/b.json 2>$O/b.err; tail -2 $O/b.err
python -c "import json;d=json.load(open('$O/b.json'));print('tail $V cqd ms/step %.2f'%d['ms_per_step'],{k:round(v,2) for k,v in d['phases_ms'].items()})"; done
PN_MGS_TAIL_VARIANT=b timeout 600 python -m pytest tests/test_fullsize.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "headline or least_squares or breakdown" 2>&1 | tail -2
