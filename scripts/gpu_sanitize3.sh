# compute-sanitizer over this session's new kernels: lookahead back
# substitutions (smem step counter + named barrier), the flow kernel with the
# hold / pick rules and ownership tables, padded TMA trees
mkdir -p gpurun_out/san3
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/san3
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "back_substitution and (look or lanes or blocked) and (77 or 31 or 64 or 33 or 300)" > $O/${tool}_bsub.log 2>&1
  echo "$tool bsub rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Race|Invalid" $O/${tool}_bsub.log | head -6
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 python -m pytest tests/test_tree_pad.py -m gpu -q -p no:cacheprovider -x -k "cqd-64 or rdd" > $O/${tool}_tree.log 2>&1
  echo "$tool tree rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Race|Invalid" $O/${tool}_tree.log | head -6
done
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 python -m pytest tests/test_flow_sched.py -m gpu -q -p no:cacheprovider -x -k "table_file" > $O/${tool}_flow.log 2>&1
  echo "$tool flow rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Race|Invalid" $O/${tool}_flow.log | head -6
done
