mkdir -p gpurun_out/fzp
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/fzp
B="python bench.py --batch 296 --dim 256 --terms 256 --base dd --steps 1 --warmup 1 --max-iters 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval_fused -s 2 -c 1 -o /tmp/prof_fz $B > /dev/null 2>$O/fz.err
ncu -i /tmp/prof_fz.ncu-rep --page details --csv > $O/fz_details.csv 2>>$O/fz.err
ncu -i /tmp/prof_fz.ncu-rep --page raw --csv > $O/fz_raw.csv 2>>$O/fz.err
ncu -i /tmp/prof_fz.ncu-rep --page source --csv 2>>$O/fz.err | gzip > $O/fz_source.csv.gz
python scripts/ncu_summary.py $O/fz_raw.csv
