mkdir -p gpurun_out/sw
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/sw
for V in warp narrow; do PN_BATCH_GROUPS=1 PN_BATCH_SLOTS=1036 PN_SOLVE_VARIANT=$V timeout 900 python bench.py --batch 1036 --dim 256 --terms 256 --base dd --steps 1 --warmup 1 --max-iters 2 > $O/c5.json 2> $O/c5.err; tail -2 $O/c5.err
python -c "import json;d=json.load(open('$O/c5.json'));print('c5 1036 slots $V', round(d['value'],1), d['roofline']['frac'])"; done
PN_BATCH_GROUPS=1 PN_BATCH_SLOTS=1036 timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active --clock-control none --csv --log-file $O/launches2.csv python bench.py --batch 1036 --dim 256 --terms 256 --base dd --steps 1 --warmup 1 --max-iters 1 > /dev/null 2>$O/launch.err
python scripts/ncu_summary.py $O/launches2.csv | head -4
