mkdir -p gpurun_out/san
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/san
SEL="test_least_squares_golden or test_evaluate_golden or test_back_substitution_vs_oracle or test_newton_c1_golden or test_residual"
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "($SEL) and (cqd or cdd or mgs_24x13 or mgs_40x17 or c1 or vec)" > $O/racecheck2.log 2>&1
echo "racecheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Race" $O/racecheck2.log | head -5
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 --error-exitcode 99 python -m pytest tests/test_batch.py -m gpu -q -p no:cacheprovider -x -k "multi_panel or slot_refill" > $O/racecheck2_batch.log 2>&1
echo "racecheck batch rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Race" $O/racecheck2_batch.log | head -5
for tool in memcheck racecheck; do timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 python -m pytest tests/test_fullsize.py -m gpu -q -p no:cacheprovider -x -k "tail_split and 1536" > $O/${tool}_tail.log 2>&1
echo "$tool tail rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Race|Invalid" $O/${tool}_tail.log | head -5; done
