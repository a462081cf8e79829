#!/bin/bash
cd "$(dirname "$0")/.."
OUT=gpurun_out/r02
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_edges.py tests/test_gpu_api.py tests/test_gpu_acceptance.py -m gpu -q -x > $OUT/pytest_small.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_small.log
timeout 300 python scripts/update_small.py 2>&1 | tee $OUT/update_small.txt
SKIP_TESTS=1 bash scripts/r02_iter.sh
