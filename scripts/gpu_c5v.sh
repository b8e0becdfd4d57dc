mkdir -p gpurun_out/c5v
O=gpurun_out/c5v
for cfg in "narrow 4" "narrow 2" "narrow 6" "wide 4" "narrow 4"; do
  set -- $cfg
  PN_SOLVE_VARIANT=$1 PN_BATCH_GROUPS=$2 timeout 900 python bench.py --batch 2048 --dim 256 --terms 256 --base dd > $O/c5.json 2>$O/c5.err
  python -c "import json; d=json.loads(open('$O/c5.json').read().strip().splitlines()[-1]); print('$1 groups $2', round(d['value']))"
done
