# C1: back substitution variants at n = 32
set -x
mkdir -p gpurun_out/c1
O=gpurun_out/c1
for b in d dd qd; do for bm in look single blocked; do
  PN_BACKSUB_MODE=$bm timeout 600 python bench.py --dim 32 --terms 32 --k 8 --base $b --steps 50 --warmup 10 --no-cpu-baseline > $O/m.json 2>$O/m.err
  python -c "import json; d=json.loads(open('$O/m.json').read().strip().splitlines()[-1]); print('$b $bm', round(d['ms_per_step'],4), round(d['e2e']['value']), d['phases_ms'], d['roofline']['seconds'])"
done; done
