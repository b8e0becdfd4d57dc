# flow kernel 1-barrier reductions (cqd step) + solve variants for C5
mkdir -p gpurun_out/it3
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/it3
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cqd.json 2>$O/bench_cqd.err; tail -3 $O/bench_cqd.err
python -c "import json;d=json.load(open('$O/bench_cqd.json'));print('cqd ms/step %.2f'%d['ms_per_step'],{k:round(v,2) for k,v in d['phases_ms'].items()})"
for V in wide narrow; do
  PN_SOLVE_VARIANT=$V timeout 900 python bench.py --batch 1184 --dim 256 --terms 256 --base dd --steps 1 --warmup 1 > $O/c5_$V.json 2> $O/c5_$V.err; tail -3 $O/c5_$V.err
  python -c "import json;d=json.load(open('$O/c5_$V.json'));print('$V', round(d['value'],1), d['roofline']['frac'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cqd.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>$O/launch.err
python scripts/ncu_summary.py $O/launches_cqd.csv
