#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
PYTEST_FILES="tests/test_gpu_f64_update.py tests/test_gpu_split.py" PYTEST_ARGS="-q --timeout 600" bash scripts/r02_tests.sh
timeout 900 python scripts/split_perf.py 2>&1 | tee gpurun_out/r02/split_perf.txt
for m in blobs gauss; do
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02/split_launches_$m.csv python scripts/split_one.py $m > /dev/null 2>&1
echo "== $m"; python scripts/launch_table.py gpurun_out/r02/split_launches_$m.csv
done
