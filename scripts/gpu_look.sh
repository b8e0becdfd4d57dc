# lookahead back substitution (cqd)
set -x
mkdir -p gpurun_out/look
O=gpurun_out/look
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "back_sub or singular" 2>&1 | tail -3
PN_BACKSUB_MODE=look timeout 900 python -m pytest tests/test_fullsize.py tests/test_acceptance_gpu.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "headline or c3 or criterion7" 2>&1 | tail -3
for m in look lanes look lanes; do
  PN_BACKSUB_MODE=$m timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('$m', d['ms_per_step'], d['backsub']['seconds'])"
done
PN_BACKSUB_MODE=look timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_backsub --csv --log-file $O/launch_look.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>$O/n.err
python scripts/ncu_summary.py $O/launch_look.csv
