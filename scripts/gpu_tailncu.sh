mkdir -p gpurun_out/tailncu
O=gpurun_out/tailncu
export PATH=/usr/local/cuda/bin:$PATH
PN_MGS_TAIL_CLUSTER=1 timeout 900 ncu --set full --clock-control none -k regex:k_mgs_tail -c 1 -o /tmp/prof_tailcl python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/out.txt 2>$O/err.txt; echo "rc=$?"
tail -5 $O/err.txt
ncu -i /tmp/prof_tailcl.ncu-rep --page raw --csv > $O/raw.csv 2>>$O/err.txt
python scripts/ncu_summary.py $O/raw.csv | head -8
PN_MGS_TAIL_CLUSTER=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_mgs_tail --csv --log-file $O/launch.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>$O/n.err
cat $O/launch.csv | tail -3
