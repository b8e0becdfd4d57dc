# padded TMA tree rows + unit-exponent buckets: parity, eval time, bank conflicts
set -x
mkdir -p gpurun_out/tpad
O=gpurun_out/tpad
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider -k "eval or c2 or batch or fused or step or golden" 2>&1 | tail -3
for pad in 1 0; do
  PN_TREE_PAD=$pad timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$pad.json 2>$O/bench_$pad.err
  PN_TREE_PAD=$pad timeout 600 python bench.py --base dd --steps 5 --warmup 3 --no-cpu-baseline > $O/benchdd_$pad.json 2>$O/benchdd_$pad.err
  PN_TREE_PAD=$pad timeout 900 python bench.py --batch 2048 --dim 256 --terms 256 --base dd > $O/c5_$pad.json 2>$O/c5_$pad.err
  for f in bench_$pad benchdd_$pad c5_$pad; do python -c "import json,sys; d=json.loads(open('$O/$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d.get('ms_per_step'), d.get('phases_ms'), d.get('eval_roofline',{}).get('seconds'))"; done
done
M=gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 600 ncu --metrics $M --clock-control none -k regex:"k_mono" --csv --log-file $O/launch_cqd.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>$O/n1.err
timeout 600 ncu --metrics $M --clock-control none -k regex:"k_mono" -c 6 --csv --log-file $O/launch_c5.csv python bench.py --batch 296 --dim 256 --terms 256 --base dd --steps 1 --warmup 1 --max-iters 2 > /dev/null 2>$O/n3.err
python scripts/ncu_summary.py $O/launch_cqd.csv $O/launch_c5.csv
