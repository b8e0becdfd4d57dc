mkdir -p gpurun_out/seg
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/seg
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -3
timeout 900 python bench.py --batch 1184 --dim 256 --terms 256 --base dd --steps 1 --warmup 1 > $O/c5.json 2> $O/c5.err; tail -3 $O/c5.err
python -c "import json;d=json.load(open('$O/c5.json'));print('c5', round(d['value'],1), d['roofline']['frac'])"
for b in qd dd d; do timeout 600 python bench.py --base $b --steps 5 --warmup 2 --no-cpu-baseline > $O/bench_c$b.json 2>$O/bench_c$b.err; tail -3 $O/bench_c$b.err;
python -c "import json;d=json.load(open('$O/bench_c$b.json'));print('c$b ms/step %.2f'%d['ms_per_step'],{k:round(v,2) for k,v in d['phases_ms'].items()})"; done
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --batch 296 --dim 256 --terms 256 --base dd --steps 1 --warmup 1 --max-iters 2 > /dev/null 2>$O/launch.err
python scripts/ncu_summary.py $O/launches.csv
