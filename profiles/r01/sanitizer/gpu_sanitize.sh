# compute-sanitizer over small parity cases of every kernel family
mkdir -p gpurun_out/san
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/san
SEL="test_least_squares_golden or test_evaluate_golden or test_back_substitution_vs_oracle or test_newton_c1_golden or test_residual"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "($SEL) and (cqd or cdd or mgs_24x13 or mgs_40x17 or c1 or vec)" > $O/$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Race|Invalid" $O/$tool.log | head -8
done
for tool in memcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 python -m pytest tests/test_batch.py tests/test_fused.py -m gpu -q -p no:cacheprovider -x -k "multi_panel or slot_refill or breakdown or fused_batch" > $O/${tool}_batch.log 2>&1
  echo "$tool batch rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Race|Invalid" $O/${tool}_batch.log | head -8
done
