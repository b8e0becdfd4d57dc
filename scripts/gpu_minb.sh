set -x
mkdir -p gpurun_out/minb
O=gpurun_out/minb
PN_TREE_MINB=3 timeout 900 python -m pytest tests/test_fullsize.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "c2 and cqd" 2>&1 | tail -2
for mb in 1 3 1 3; do
  PN_TREE_MINB=$mb timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/m.json 2>$O/m.err
  python -c "import json; d=json.loads(open('$O/m.json').read().strip().splitlines()[-1]); print('minb $mb', round(d['ms_per_step'],3), d['phases_ms']['evaluate'])"
done
