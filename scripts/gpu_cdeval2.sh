mkdir -p gpurun_out/cdeval
O=gpurun_out/cdeval
PN_TREE_MINB=8 timeout 900 python -m pytest tests/test_fullsize.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "c2 and cd" > $O/t.log 2>&1; tail -1 $O/t.log
for cfg in "1 0" "6 0" "8 0" "1 1" "8 1"; do
  set -- $cfg
  PN_TREE_MINB=$1 PN_TREE_TMA=$2 timeout 600 python bench.py --base d --steps 10 --warmup 3 --no-cpu-baseline > $O/b.json 2>$O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); e=d['eval_roofline']; print('minb $1 tma $2', round(d['ms_per_step'],3), round(e['seconds']*1e3,3), round(e['achieved_gbs']))"
done
