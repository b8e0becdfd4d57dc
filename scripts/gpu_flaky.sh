mkdir -p gpurun_out/flaky
O=gpurun_out/flaky
for i in 1 2; do
  timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $O/full_$i.log 2>&1; echo "full $i: $(tail -1 $O/full_$i.log)"
done
for i in 1 2 3 4 5; do
  timeout 900 python -m pytest tests/test_flow_sched.py tests/test_fullsize.py tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "flow or tail or back_sub or headline or least_squares_vs_oracle" > $O/rep_$i.log 2>&1; echo "rep $i: $(tail -1 $O/rep_$i.log)"
done
