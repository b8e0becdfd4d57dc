export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out/flow2
O=gpurun_out/flow2
PN_FLOW_NT=512 timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -p no:cacheprovider -x -k "least_squares or breakdown" 2>&1 | tail -2
for V in 512 256; do PN_FLOW_NT=$V timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cqd_$V.json 2>$O/bench_cqd.err; tail -3 $O/bench_cqd.err
python -c "import json;d=json.load(open('$O/bench_cqd_$V.json'));print('NT=$V cqd ms/step %.2f'%d['ms_per_step'],{k:round(v,2) for k,v in d['phases_ms'].items()})"; done
