# batched C5 path: parity tests + bench at a few widths
mkdir -p gpurun_out/batch
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/batch
timeout 900 python -m pytest tests/test_batch.py -m gpu -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -15
for B in ${BATCHES:-64 592}; do
  timeout 900 python bench.py --batch $B --dim 256 --terms 256 --base dd --steps 1 --warmup 1 > $O/c5_$B.json 2> $O/c5_$B.err; tail -3 $O/c5_$B.err; cat $O/c5_$B.json; echo
done
