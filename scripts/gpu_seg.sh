mkdir -p gpurun_out/segm
O=gpurun_out/segm
for b in qd dd d; do for sm in 1 4 6; do
  PN_SEG_MINB=$sm timeout 600 python bench.py --base $b --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('$b seg minb $sm', round(d['ms_per_step'],3), round(d['phases_ms']['evaluate'],3))"
done; done
PN_SEG_MINB=6 timeout 900 python -m pytest tests/test_fullsize.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "c2" > $O/t.log 2>&1; tail -1 $O/t.log
