# round evidence: benches (default, reference arm, levels, C4, C5), launch
# lists with DRAM bytes, full ncu captures of the top kernels
set -x
mkdir -p gpurun_out/ev
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/ev
nproc
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; cat $O/bench_default.json
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; cat $O/bench_reference.json
for b in dd d; do timeout 600 python bench.py --base $b --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c$b.json 2>$O/bench_c$b.err; done
timeout 900 python bench.py --converge --max-iters 10 > $O/c4_square.json 2>$O/c4_square.err
timeout 900 python bench.py --converge --rows 1536 --max-iters 10 > $O/c4_over.json 2>$O/c4_over.err
timeout 900 python bench.py --batch 2048 --dim 256 --terms 256 --base dd > $O/c5_2048.json 2>$O/c5_2048.err; cat $O/c5_2048.json
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file $O/launches_cqd.csv $B > /dev/null 2>$O/launch.err
for spec in "mgs:k_mgs_flow" "tree:k_mono_tree" "seg:k_segments" "bsub:k_backsub" "tail:k_mgs_tail"; do
  name=${spec%%:*}; kern=${spec#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kern -c 1 -o /tmp/prof_$name $B > /dev/null 2>$O/$name.err
  ncu -i /tmp/prof_$name.ncu-rep --page details --csv > $O/${name}_details.csv 2>>$O/$name.err
  ncu -i /tmp/prof_$name.ncu-rep --page raw --csv > $O/${name}_raw.csv 2>>$O/$name.err
done
BD="python bench.py --base dd --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file $O/launches_cdd.csv $BD > /dev/null 2>$O/launchd.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mgs_pipe -c 1 -o /tmp/prof_pipe $BD > /dev/null 2>$O/pipe.err
ncu -i /tmp/prof_pipe.ncu-rep --page details --csv > $O/pipe_details.csv 2>>$O/pipe.err
ncu -i /tmp/prof_pipe.ncu-rep --page raw --csv > $O/pipe_raw.csv 2>>$O/pipe.err
C5="python bench.py --batch 296 --dim 256 --terms 256 --base dd --steps 1 --warmup 1 --max-iters 2"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file $O/launches_c5.csv $C5 > /dev/null 2>$O/launch5.err
timeout 900 ncu --set full --clock-control none -k regex:k_solve_batch -s 1 -c 1 -o /tmp/prof_solve $C5 > /dev/null 2>$O/solve.err
ncu -i /tmp/prof_solve.ncu-rep --page details --csv > $O/solve_details.csv 2>>$O/solve.err
ncu -i /tmp/prof_solve.ncu-rep --page raw --csv > $O/solve_raw.csv 2>>$O/solve.err
python scripts/ncu_summary.py $O/launches_cqd.csv $O/launches_cdd.csv $O/launches_c5.csv $O/mgs_raw.csv $O/tree_raw.csv $O/seg_raw.csv $O/bsub_raw.csv $O/tail_raw.csv $O/pipe_raw.csv $O/solve_raw.csv > $O/summary.txt 2>&1
du -sh gpurun_out
