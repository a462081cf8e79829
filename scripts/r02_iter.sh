#!/bin/bash
# GPU tests + per-config iteration timing + a launch list of 3 pipelined iterations per config.
cd "$(dirname "$0")/.."
OUT=gpurun_out/r02
mkdir -p $OUT
if [ -z "${SKIP_TESTS:-}" ]; then
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 $OUT/pytest_gpu.log
fi
timeout 600 python scripts/config_perf.py 2>&1 | tee $OUT/config_perf.txt
for c in 4 2; do
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/iter_launches_cfg$c.csv python scripts/iter_launches.py $c 3 > /dev/null 2>&1
echo "== config $c launches (3 iterations)"; python scripts/launch_table.py $OUT/iter_launches_cfg$c.csv
done
