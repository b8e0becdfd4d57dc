mkdir -p gpurun_out/warp
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/warp
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -4
for b in dd d; do for mode in warp dataflow; do PN_MGS_MODE=$mode timeout 600 python bench.py --base $b --steps 5 --warmup 2 --no-cpu-baseline > $O/bench_c${b}_$mode.json 2>$O/bench_c$b.err; tail -3 $O/bench_c$b.err;
python -c "import json;d=json.load(open('$O/bench_c${b}_$mode.json'));print('c$b $mode ms/step %.2f'%d['ms_per_step'],{k:round(v,2) for k,v in d['phases_ms'].items()})"; done; done
