mkdir -p gpurun_out/fz
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/fz
timeout 900 python -m pytest tests/test_fused.py tests/test_batch.py -m gpu -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -15
for V in 1 0; do
  PN_EVAL_FUSED=$V timeout 900 python bench.py --batch 1184 --dim 256 --terms 256 --base dd --steps 1 --warmup 1 > $O/c5_f$V.json 2> $O/c5_f$V.err; tail -3 $O/c5_f$V.err
  python -c "import json;d=json.load(open('$O/c5_f$V.json'));print('fused=$V', round(d['value'],1), d['roofline']['frac'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file $O/launches.csv python bench.py --batch 296 --dim 256 --terms 256 --base dd --steps 1 --warmup 1 --max-iters 2 > /dev/null 2>$O/launch.err
python scripts/ncu_summary.py $O/launches.csv
