#!/bin/bash
# Full GPU suite, then per-config timing (scripts/config_perf.py) and the
# end-of-iteration kernel timings (scripts/norm_tail_perf.py).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS:-} > gpurun_out/r02/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02/pytest_gpu.log
timeout 300 python scripts/norm_tail_perf.py 2>&1 | tail -2
timeout 600 python scripts/config_perf.py 2>&1 | tail -4
