#!/bin/bash
# Round evidence: GPU suite + smoke, benches (default line, reference arm,
# C4, families), launch lists with DRAM bytes, full ncu captures of the top
# kernels of each level, summaries.  Output: gpurun_out/ev (scratch) ->
# copied to profiles/<round>/ by hand.
set -x
mkdir -p gpurun_out/ev
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/ev
nproc
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 2400 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 python bench.py --converge --max-iters 10 > $O/c4_square.json 2>$O/c4_square.err
timeout 900 python bench.py --converge --rows 1536 --max-iters 10 > $O/c4_over.json 2>$O/c4_over.err
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extras --e2e-steps 1"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/launches_cqd.csv $B > /dev/null 2>$O/launch.err
for spec in "mgs:k_mgs_flow" "tree:k_mono_tree" "seg:k_segments" "bsub:k_backsub" "tail:k_mgs_tail"; do
  name=${spec%%:*}; kern=${spec#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kern -c 1 -o /tmp/prof_$name $B > /dev/null 2>$O/$name.err
  ncu -i /tmp/prof_$name.ncu-rep --page details --csv > $O/${name}_details.csv 2>>$O/$name.err
  ncu -i /tmp/prof_$name.ncu-rep --page raw --csv > $O/${name}_raw.csv 2>>$O/$name.err
done
for lv in dd d; do
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/launches_c$lv.csv $B --base $lv > /dev/null 2>$O/launch$lv.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mgs_pipe -c 1 -o /tmp/prof_pipe $B --base dd > /dev/null 2>$O/pipe.err
ncu -i /tmp/prof_pipe.ncu-rep --page details --csv > $O/pipe_details.csv 2>>$O/pipe.err
ncu -i /tmp/prof_pipe.ncu-rep --page raw --csv > $O/pipe_raw.csv 2>>$O/pipe.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval_rows -c 1 -o /tmp/prof_rows $B --base d > /dev/null 2>$O/rows.err
ncu -i /tmp/prof_rows.ncu-rep --page details --csv > $O/rows_details.csv 2>>$O/rows.err
ncu -i /tmp/prof_rows.ncu-rep --page raw --csv > $O/rows_raw.csv 2>>$O/rows.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mgs_pipe -c 1 -o /tmp/prof_piped $B --base d > /dev/null 2>$O/piped.err
ncu -i /tmp/prof_piped.ncu-rep --page raw --csv > $O/piped_raw.csv 2>>$O/piped.err
C5="python bench.py --batch 296 --dim 256 --terms 256 --base dd --steps 1 --warmup 1 --max-iters 2"
timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/launches_c5.csv $C5 > /dev/null 2>$O/launch5.err
timeout 900 ncu --set full --clock-control none -k regex:k_solve_batch -s 1 -c 1 -o /tmp/prof_solve $C5 > /dev/null 2>$O/solve.err
ncu -i /tmp/prof_solve.ncu-rep --page raw --csv > $O/solve_raw.csv 2>>$O/solve.err
CY="python bench.py --family cyclic --base qd --dim 448 --steps 1 --warmup 1"
timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/launches_cyclic_qd448.csv $CY > /dev/null 2>$O/launchcy.err
timeout 900 ncu --set full --clock-control none -k regex:k_mono_warp -c 1 -o /tmp/prof_warp $CY > /dev/null 2>$O/warp.err
ncu -i /tmp/prof_warp.ncu-rep --page raw --csv > $O/warp_raw.csv 2>>$O/warp.err
python scripts/ncu_summary.py $O/launches_cqd.csv $O/launches_cdd.csv $O/launches_cd.csv $O/launches_c5.csv $O/launches_cyclic_qd448.csv $O/mgs_raw.csv $O/tree_raw.csv $O/seg_raw.csv $O/bsub_raw.csv $O/tail_raw.csv $O/pipe_raw.csv $O/piped_raw.csv $O/rows_raw.csv $O/solve_raw.csv $O/warp_raw.csv > $O/summary.txt 2>&1
du -sh gpurun_out
