mkdir -p gpurun_out/tail
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/tail
for RQ in 256 512; do PN_MGS_TAIL_RQ=$RQ PN_MGS_TRACE=$O/trace_rq$RQ.txt timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > $O/b.json 2>$O/b.err; tail -2 $O/b.err
python -c "import json;d=json.load(open('$O/b.json'));print('rq=$RQ cqd ms/step %.2f'%d['ms_per_step'],{k:round(v,2) for k,v in d['phases_ms'].items()})"; done
PN_MGS_TAIL_RQ=512 timeout 600 python -m pytest tests/test_fullsize.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "headline or c3 or least_squares" 2>&1 | tail -2
