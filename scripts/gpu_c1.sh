# config C1 (dim 32, 32 monomials of 8 vars, cd): step latency and launches
set -x
mkdir -p gpurun_out/c1
O=gpurun_out/c1
for b in d dd qd; do
  timeout 600 python bench.py --dim 32 --terms 32 --k 8 --base $b --steps 50 --warmup 10 > $O/c1_$b.json 2>$O/c1_$b.err
  python -c "import json; d=json.loads(open('$O/c1_$b.json').read().strip().splitlines()[-1]); print('$b', d['ms_per_step'], d['e2e'], d['gpu_launches'], d['phases_ms'], d.get('cpu_baseline',{}) and d['cpu_baseline']['value'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_c1.csv python bench.py --dim 32 --terms 32 --k 8 --base d --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>$O/n.err
python scripts/ncu_summary.py $O/launch_c1.csv
