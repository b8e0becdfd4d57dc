mkdir -p gpurun_out/cdeval
O=gpurun_out/cdeval
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active,lts__t_bytes.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:"k_mono|k_seg|k_power|k_zero" --csv --log-file $O/launch_cd.csv python bench.py --base d --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>$O/n.err
python scripts/ncu_summary.py $O/launch_cd.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mono_tree -c 1 -o /tmp/prof_cdtree python bench.py --base d --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>$O/f.err
ncu -i /tmp/prof_cdtree.ncu-rep --page raw --csv > $O/cdtree_raw.csv 2>>$O/f.err
ncu -i /tmp/prof_cdtree.ncu-rep --page details --csv > $O/cdtree_details.csv 2>>$O/f.err
python scripts/ncu_summary.py $O/cdtree_raw.csv
