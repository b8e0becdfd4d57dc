set -x
mkdir -p gpurun_out/minb
O=gpurun_out/minb
timeout 900 python -m pytest tests/test_fullsize.py tests/test_batch.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "c2 or c5 or multi_panel" 2>&1 | tail -2
PN_TREE_MINB=4 timeout 900 python -m pytest tests/test_fullsize.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "c2" 2>&1 | tail -2
for mb in 1 3 4; do
  PN_TREE_MINB=$mb timeout 600 python bench.py --base dd --steps 5 --warmup 3 --no-cpu-baseline > $O/m.json 2>$O/m.err
  python -c "import json; d=json.loads(open('$O/m.json').read().strip().splitlines()[-1]); print('cdd minb $mb', round(d['ms_per_step'],3), d['phases_ms']['evaluate'])"
  PN_TREE_MINB=$mb timeout 900 python bench.py --batch 2048 --dim 256 --terms 256 --base dd > $O/c5.json 2>$O/c5.err
  python -c "import json; d=json.loads(open('$O/c5.json').read().strip().splitlines()[-1]); print('c5 minb $mb', d['value'])"
done
PN_TREE_MINB=4 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/m.json 2>$O/m.err
python -c "import json; d=json.loads(open('$O/m.json').read().strip().splitlines()[-1]); print('cqd minb 4', round(d['ms_per_step'],3), d['phases_ms']['evaluate'])"
