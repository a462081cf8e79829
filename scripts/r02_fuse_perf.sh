#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
for f in 1 0; do echo "== FK_ASSIGN_FUSE=$f"; FK_ASSIGN_FUSE=$f timeout 300 python scripts/config_perf.py 2>&1 | grep cfg4; done | tee gpurun_out/r02/fuse_ab.txt
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02/iter_launches_cfg4_fused.csv python scripts/iter_launches.py 4 3 > /dev/null 2>&1
echo "== config 4 launches (3 iterations, fused)"; python scripts/launch_table.py gpurun_out/r02/iter_launches_cfg4_fused.csv
