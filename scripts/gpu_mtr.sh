mkdir -p gpurun_out/mtr
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/mtr
timeout 1200 python -m pytest tests/test_batch.py tests/test_fullsize.py -m gpu -q --timeout 600 -p no:cacheprovider -x -k "not headline" 2>&1 | tail -2
for i in 1 2; do timeout 900 python bench.py --batch 2048 --dim 256 --terms 256 --base dd --steps 1 --warmup 1 > $O/c5.json 2> $O/c5.err; tail -2 $O/c5.err
python -c "import json;d=json.load(open('$O/c5.json'));print('c5', round(d['value'],1), d['roofline']['frac'])"; done
