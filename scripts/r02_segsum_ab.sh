#!/bin/bash
# A/B: segment-chained k_segsum2 (default) vs the per-segment k_segsum
# (FK_SEGSUM_SEQ=1); update-path tests first, then configs 2/3/4, alternating.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
timeout 900 python -m pytest -x -q tests/test_gpu_kernels.py tests/test_gpu_f64_update.py tests/test_gpu_acceptance.py \
  tests/test_gpu_sharded.py tests/test_gpu_api.py > gpurun_out/r02/segsum_tests.log 2>&1; tail -3 gpurun_out/r02/segsum_tests.log
for v in 0 1 0 1; do
  echo "== FK_SEGSUM_SEQ=$v"
  FK_SEGSUM_SEQ=$v timeout 300 python scripts/config_perf.py
done > gpurun_out/r02/segsum_ab.txt 2>&1
cat gpurun_out/r02/segsum_ab.txt
