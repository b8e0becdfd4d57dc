set -x
mkdir -p gpurun_out/bstage
O=gpurun_out/bstage
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_mgs_small.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "back_sub or singular or small" 2>&1 | tail -2
for cfg in "dd 1024 1024 32" "d 1024 1024 32" "d 32 32 8" "dd 32 32 8"; do
  set -- $cfg
  timeout 600 python bench.py --base $1 --dim $2 --terms $3 --k $4 --steps 10 --warmup 3 --no-cpu-baseline > $O/m.json 2>$O/m.err
  python -c "import json; d=json.loads(open('$O/m.json').read().strip().splitlines()[-1]); print('$cfg', round(d['ms_per_step'],4), d['backsub']['seconds'], d['phases_ms'])"
done
