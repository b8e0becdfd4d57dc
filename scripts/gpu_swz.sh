# flow-kernel smem swizzle: parity, step time, bank conflicts of the MGS kernels
set -x
mkdir -p gpurun_out/swz
O=gpurun_out/swz
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "mgs or least or tail or headline or step" 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench.json 2>$O/bench.err; cat $O/bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phases_ms'], d['roofline']['frac'], d['roofline']['seconds'])"
M=gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 600 ncu --metrics $M --clock-control none -k regex:"k_mgs|k_mono|k_back|k_seg" --csv --log-file $O/cqd.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>$O/n1.err
timeout 600 ncu --metrics $M --clock-control none -k regex:"k_mgs|k_mono|k_back|k_seg" --csv --log-file $O/cdd.csv python bench.py --base dd --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>$O/n2.err
timeout 600 ncu --metrics $M --clock-control none -k regex:"k_solve|k_mono" -c 6 --csv --log-file $O/c5.csv python bench.py --batch 296 --dim 256 --terms 256 --base dd --steps 1 --warmup 1 --max-iters 2 > /dev/null 2>$O/n3.err
python scripts/ncu_summary.py $O/cqd.csv $O/cdd.csv $O/c5.csv
