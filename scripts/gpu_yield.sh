export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out/y; O=gpurun_out/y
for Y in "" 0.6 0.4 0.25; do PN_FLOW_YIELD=$Y timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > $O/b.json 2>$O/b.err; tail -2 $O/b.err
python -c "import json;d=json.load(open('$O/b.json'));print('yield=$Y cqd ms/step %.2f'%d['ms_per_step'],{k:round(v,2) for k,v in d['phases_ms'].items()})"; done
PN_FLOW_YIELD=0.4 timeout 900 python -m pytest tests/test_fullsize.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "headline or (least_squares and cqd) or breakdown" 2>&1 | tail -2
