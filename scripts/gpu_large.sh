#!/bin/bash
# large-k trees: parity (configs with k > 32) and the cyclic family timing, warp vs CTA per monomial
cd "$(dirname "$0")/.."
T=${TAG:-r02o}
timeout 1200 python -m pytest tests/test_config_parity.py tests/test_acceptance_gpu.py tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "large or cyclic or criterion or wide or k32 or eval" > gpurun_out/${T}_large_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_large_tests.log
for w in 1 0; do for b in d dd qd; do
  PN_LARGE_WARP=$w timeout 600 python bench.py --family cyclic --base $b --steps 3 --warmup 1 > gpurun_out/${T}_cyc_${b}_w$w.json 2>&1
done; done
tail -3 gpurun_out/${T}_large_tests.log
