mkdir -p gpurun_out/c4
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/c4
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -p no:cacheprovider -x -k "least_squares or breakdown" 2>&1 | tail -3
timeout 900 python bench.py --converge --rows 1536 --max-iters 10 > $O/c4_over.json 2>$O/c4_over.err; tail -3 $O/c4_over.err; cat $O/c4_over.json; echo
