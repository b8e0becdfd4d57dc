# round-end style check: tests, smoke, default bench (driver invocation), reference arm, C5 batch
mkdir -p gpurun_out/full
export PATH=/usr/local/cuda/bin:$PATH
nproc; python -c "import os; print('cpu_count', os.cpu_count())"
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider 2>&1 | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/full/bench_default.json 2> gpurun_out/full/bench_default.err; tail -2 gpurun_out/full/bench_default.err; cat gpurun_out/full/bench_default.json
timeout 900 python bench.py --impl reference > gpurun_out/full/bench_reference.json 2> gpurun_out/full/bench_reference.err; tail -2 gpurun_out/full/bench_reference.err; cat gpurun_out/full/bench_reference.json
timeout 900 python bench.py --batch ${BATCH:-64} --dim 256 --terms 256 --base dd > gpurun_out/full/bench_c5.json 2> gpurun_out/full/bench_c5.err; tail -3 gpurun_out/full/bench_c5.err; cat gpurun_out/full/bench_c5.json
