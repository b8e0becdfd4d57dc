mkdir -p gpurun_out/c4
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/c4
timeout 900 python bench.py --converge --max-iters 10 > $O/c4_square.json 2>$O/c4_square.err; tail -3 $O/c4_square.err; cat $O/c4_square.json; echo
timeout 900 python bench.py --converge --rows 1536 --max-iters 10 > $O/c4_over.json 2>$O/c4_over.err; tail -3 $O/c4_over.err; cat $O/c4_over.json; echo
