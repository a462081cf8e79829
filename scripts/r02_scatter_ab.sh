#!/bin/bash
# Stable scatter: warp-table kernel vs block radix sort, correctness first.
cd "$(dirname "$0")/.."
OUT=gpurun_out/r02
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_edges.py tests/test_gpu_api.py -m gpu -q -x > $OUT/pytest_sort.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_sort.log
for m in 0 1; do echo "FK_SCATTER_RADIX=$m"; FK_SCATTER_RADIX=$m timeout 300 python scripts/update_small.py; done 2>&1 | tee $OUT/scatter_ab.txt
SHAPE=0,1,4 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_hist|k_colscan|k_scan|k_scatter|k_segsum' \
  --csv --log-file $OUT/update_launches.csv python scripts/update_small.py > /dev/null 2>&1
