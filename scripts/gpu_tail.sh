mkdir -p gpurun_out/tail
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/tail
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -p no:cacheprovider -x -k "least_squares or breakdown or newton" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_fullsize.py -m gpu -q -p no:cacheprovider -x -k "headline or c3" 2>&1 | tail -2
for V in "" 0 32 148; do PN_MGS_TAIL=$V PN_MGS_TRACE=$O/trace_$V.txt timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > $O/b.json 2>$O/b.err; tail -2 $O/b.err
python -c "import json;d=json.load(open('$O/b.json'));print('tail=$V cqd ms/step %.2f'%d['ms_per_step'],{k:round(v,2) for k,v in d['phases_ms'].items()})"; done
PN_MGS_TAIL= timeout 600 python bench.py --rows 1536 --steps 3 --warmup 2 --no-cpu-baseline > $O/b.json 2>$O/b.err; python -c "import json;d=json.load(open('$O/b.json'));print('over cqd ms/step %.2f'%d['ms_per_step'],{k:round(v,2) for k,v in d['phases_ms'].items()})"
