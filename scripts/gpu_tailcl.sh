mkdir -p gpurun_out/tailcl
O=gpurun_out/tailcl
PN_MGS_TAIL_CLUSTER=1 timeout 900 python -m pytest tests/test_fullsize.py tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "tail or headline or (least_squares_vs_oracle and cqd) or (breakdown and qd)" > $O/t.log 2>&1; tail -1 $O/t.log; grep -m2 "refused" $O/t.log
for c in 0 1 0 1; do
  PN_MGS_TAIL_CLUSTER=$c timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('cluster $c', round(d['ms_per_step'],2), round(d['roofline']['seconds']*1e3,2))"; grep -m1 refused $O/b.err
done
PN_MGS_TAIL_CLUSTER=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_mgs_tail --csv --log-file $O/launch.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>$O/n.err
python scripts/ncu_summary.py $O/launch.csv
