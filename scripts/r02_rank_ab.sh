#!/bin/bash
# stable scatter ranks: warp bitonic sort (default) vs returning atomics (A/B) + update/argsort tests
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
PYTEST_FILES="tests/test_gpu_kernels.py tests/test_gpu_acceptance.py tests/test_gpu_api.py tests/test_gpu_stream_files.py" PYTEST_ARGS="-q -x" bash scripts/r02_tests.sh
for v in sort atomic; do echo "== FK_SCATTER_RANK=$v"; FK_SCATTER_RANK=$v timeout 300 python scripts/config_perf.py 2>&1 | grep -E "cfg2|cfg3|cfg4 B"; done
