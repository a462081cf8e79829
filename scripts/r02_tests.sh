#!/bin/bash
# GPU test suite only (log under gpurun_out/r02/).
cd "$(dirname "$0")/.."
OUT=gpurun_out/r02
mkdir -p $OUT
timeout 1500 python -m pytest ${PYTEST_FILES:-tests} -m gpu -q -x ${PYTEST_ARGS:-} > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 $OUT/pytest_gpu.log
