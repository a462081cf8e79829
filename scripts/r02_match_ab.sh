#!/bin/bash
# Warp scatter ranks by match.any without atomics (FK_SCATTER_RANK=match) vs returning shared atomics:
# stability/parity tests with the switch on, then per-config update timings on one box.
cd "$(dirname "$0")/.."
FK_SCATTER_RANK=match timeout 900 python -m pytest -q -x tests/test_gpu_kernels.py tests/test_gpu_api.py -m gpu 2>&1 | tail -2
for r in 1 2; do
  for v in atomic match; do
    echo "== FK_SCATTER_RANK=$v"
    FK_SCATTER_RANK=$v timeout 600 python scripts/config_perf.py 2>&1 | sed -n 1,5p | cut -c1-200
  done
done
