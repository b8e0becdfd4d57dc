mkdir -p gpurun_out/sw
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/sw
timeout 1200 python -m pytest tests/test_batch.py tests/test_fused.py -m gpu -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -3
for V in warp narrow; do PN_SOLVE_VARIANT=$V timeout 900 python bench.py --batch 2048 --dim 256 --terms 256 --base dd --steps 1 --warmup 1 > $O/c5.json 2> $O/c5.err; tail -2 $O/c5.err
python -c "import json;d=json.load(open('$O/c5.json'));print('c5 $V', round(d['value'],1), d['roofline']['frac'])"; done
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active --clock-control none --csv --log-file $O/launches.csv python bench.py --batch 296 --dim 256 --terms 256 --base dd --steps 1 --warmup 1 --max-iters 2 > /dev/null 2>$O/launch.err
python scripts/ncu_summary.py $O/launches.csv | head -5
