#!/bin/bash
# Stable-scatter A/B (ballot vs match.any) + launch list + one full ncu capture per shape.
cd "$(dirname "$0")/.."
OUT=gpurun_out/r02
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -k "argsort or deterministic or update" > $OUT/pytest_sort.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_sort.log
for m in 0 1; do echo "FK_SCATTER_MATCH=$m"; FK_SCATTER_MATCH=$m timeout 300 python scripts/update_small.py; done 2>&1 | tee $OUT/scatter_ab.txt
SHAPE=0,1,4 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_hist|k_colscan|k_scan|k_scatter|k_segsum' \
  --csv --log-file $OUT/update_launches.csv python scripts/update_small.py > /dev/null 2>&1
for sh in 1 4; do
SHAPE=$sh timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scatter_stable -s 3 -c 1 \
  -o $OUT/scatter_shape$sh -f python scripts/update_small.py > /dev/null 2>&1; echo "ncu shape $sh rc=$?"
done
