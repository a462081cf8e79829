#!/bin/bash
# Programmatic dependent launch in the update chain (FK_PDL=1: scatter -> segsum -> normalize tail):
# parity tests with the switch on, then per-config timings (same box, alternating).
cd "$(dirname "$0")/.."
FK_PDL=1 timeout 900 python -m pytest -q -x tests/test_gpu_kernels.py tests/test_gpu_api.py tests/test_gpu_acceptance.py -m gpu 2>&1 | tail -2
for r in 1 2 3; do
  for v in 0 1; do
    echo "== FK_PDL=$v"
    FK_PDL=$v timeout 600 python scripts/config_perf.py 2>&1 | sed -n 1,5p | cut -c1-130
  done
done
