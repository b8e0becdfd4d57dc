mkdir -p gpurun_out/var2
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/var2
for lib in paper_1402_2626_b200/lib/libpolynewt_b200.so paper_1402_2626_b200/lib/libpolynewt_b200_g8.so; do
  PN_LIB=$lib timeout 600 python bench.py --base dd --steps 5 --warmup 2 --no-cpu-baseline > $O/cdd.json 2>$O/cdd.err
  python -c "import json;d=json.load(open('$O/cdd.json'));print('$lib cdd ms/step %.2f'%d['ms_per_step'],{k:round(v,2) for k,v in d['phases_ms'].items()})"
  PN_LIB=$lib timeout 900 python bench.py --batch 1184 --dim 256 --terms 256 --base dd --steps 1 --warmup 1 > $O/c5.json 2> $O/c5.err
  python -c "import json;d=json.load(open('$O/c5.json'));print('$lib c5', round(d['value'],1), d['roofline']['frac'])"
done
for b in dd d; do for mode in flow dataflow; do PN_MGS_MODE=$mode timeout 600 python bench.py --base $b --steps 5 --warmup 2 --no-cpu-baseline > $O/b.json 2>$O/b.err
python -c "import json;d=json.load(open('$O/b.json'));print('c$b $mode ms/step %.2f'%d['ms_per_step'],{k:round(v,2) for k,v in d['phases_ms'].items()})"; done; done
