mkdir -p gpurun_out/bs
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/bs
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -p no:cacheprovider -x -k "back_substitution or singular or newton or least_squares_golden" 2>&1 | tail -2
for b in dd qd; do for V in lanes blocked; do PN_BACKSUB_MODE=$V timeout 600 python bench.py --base $b --steps 5 --warmup 2 --no-cpu-baseline > $O/b.json 2>$O/b.err; tail -2 $O/b.err
python -c "import json;d=json.load(open('$O/b.json'));print('c$b $V ms/step %.2f'%d['ms_per_step'], 'bsub', round(d['backsub']['seconds']*1e3,3))"; done; done
