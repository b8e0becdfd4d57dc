mkdir -p gpurun_out/n3
O=gpurun_out/n3
PN_SOLVE_VARIANT=n3 timeout 1500 python -m pytest tests/test_batch.py tests/test_fullsize.py -m gpu -q -x --timeout 900 -p no:cacheprovider -k "batch or c5" > $O/t.log 2>&1; tail -1 $O/t.log
for v in narrow n3 narrow n3; do
PN_SOLVE_VARIANT=$v timeout 900 python bench.py --batch 2048 --dim 256 --terms 256 --base dd > $O/c5.json 2>$O/c5.err
python -c "import json; d=json.loads(open('$O/c5.json').read().strip().splitlines()[-1]); print('c5 $v', d['value'])"
done
