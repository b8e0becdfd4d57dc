# lookahead back substitution, all levels
set -x
mkdir -p gpurun_out/look2
O=gpurun_out/look2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "back_sub or singular or least" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_fullsize.py tests/test_acceptance_gpu.py -m gpu -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -3
for b in dd d; do for m in look blocked; do
  PN_BACKSUB_MODE=$m timeout 600 python bench.py --base $b --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('$b $m', d['ms_per_step'], d['backsub']['seconds'])"
done; done
