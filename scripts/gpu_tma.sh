mkdir -p gpurun_out/tma
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/tma
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -2
for V in 1 0; do for b in qd dd d; do PN_TREE_TMA=$V timeout 600 python bench.py --base $b --steps 5 --warmup 2 --no-cpu-baseline > $O/b.json 2>$O/b.err; tail -2 $O/b.err
python -c "import json;d=json.load(open('$O/b.json'));print('tma=$V c$b ms/step %.2f'%d['ms_per_step'],{k:round(v,2) for k,v in d['phases_ms'].items()})"; done
PN_TREE_TMA=$V timeout 900 python bench.py --batch 1184 --dim 256 --terms 256 --base dd --steps 1 --warmup 1 > $O/c5.json 2> $O/c5.err; tail -2 $O/c5.err
python -c "import json;d=json.load(open('$O/c5.json'));print('tma=$V c5', round(d['value'],1), d['roofline']['frac'])"; done
