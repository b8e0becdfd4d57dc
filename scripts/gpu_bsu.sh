# back substitution: unrolled update loops
set -x
mkdir -p gpurun_out/bsu
O=gpurun_out/bsu
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "back or least or headline or c3 or solve" 2>&1 | tail -3
for b in qd dd d; do for u in 1 0; do
  PN_BACKSUB_UNROLL=$u timeout 600 python bench.py --base $b --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('$b unroll $u', d['ms_per_step'], d['backsub'])"
done; done
