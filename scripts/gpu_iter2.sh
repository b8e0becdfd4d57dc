# parity tests, default bench, C5 bench, backsub check
mkdir -p gpurun_out/it2
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/it2
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -4
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cqd.json 2>$O/bench_cqd.err; tail -3 $O/bench_cqd.err
python -c "import json;d=json.load(open('$O/bench_cqd.json'));print('cqd ms/step %.2f'%d['ms_per_step'],{k:round(v,2) for k,v in d['phases_ms'].items()})"
for B in ${BATCHES:-592 2048}; do
  timeout 900 python bench.py --batch $B --dim 256 --terms 256 --base dd --steps 1 --warmup 1 > $O/c5_$B.json 2> $O/c5_$B.err; tail -3 $O/c5_$B.err; cat $O/c5_$B.json; echo
done
