export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out/m2; O=gpurun_out/m2
for lib in paper_1402_2626_b200/lib/libpolynewt_b200.so paper_1402_2626_b200/lib/libpolynewt_b200_m2.so; do for b in dd d; do
PN_LIB=$lib timeout 600 python bench.py --base $b --steps 5 --warmup 2 --no-cpu-baseline > $O/b.json 2>$O/b.err; tail -2 $O/b.err
python -c "import json;d=json.load(open('$O/b.json'));print('$lib c$b ms/step %.2f'%d['ms_per_step'],{k:round(v,2) for k,v in d['phases_ms'].items()})"; done; done
