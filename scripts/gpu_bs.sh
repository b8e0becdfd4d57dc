mkdir -p gpurun_out/bs
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/bs
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -3
for V in lanes blocked; do PN_BACKSUB_MODE=$V timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cqd_$V.json 2>$O/bench_cqd.err; tail -3 $O/bench_cqd.err
python -c "import json;d=json.load(open('$O/bench_cqd_$V.json'));print('$V cqd ms/step %.2f'%d['ms_per_step'],{k:round(v,2) for k,v in d['phases_ms'].items()})"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>$O/launch.err
python scripts/ncu_summary.py $O/launches.csv | head -6
