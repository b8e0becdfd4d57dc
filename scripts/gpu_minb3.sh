mkdir -p gpurun_out/minb
O=gpurun_out/minb
timeout 1500 python -m pytest tests/test_fullsize.py tests/test_batch.py tests/test_tree_pad.py tests/test_gpu_parity.py -m gpu -q -x --timeout 900 -p no:cacheprovider -k "c2 or c5 or batch or pad or evaluat or golden" > $O/t.log 2>&1; tail -1 $O/t.log
for i in 1 2; do
timeout 900 python bench.py --batch 2048 --dim 256 --terms 256 --base dd > $O/c5.json 2>$O/c5.err
python -c "import json; d=json.loads(open('$O/c5.json').read().strip().splitlines()[-1]); print('c5', d['value'])"
done
