#!/bin/bash
# ncu --set full of the config-2 segsum and scatter (one pipelined iteration)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
timeout 600 ncu --profile-from-start off -k "regex:k_segsum|k_scatter_warp" -c 2 --set full \
  --import-source on --clock-control none -o gpurun_out/r02/prof_cfg2_update -f python scripts/iter_launches.py 2 1 \
  > gpurun_out/r02/prof_cfg2_update.log 2>&1
tail -2 gpurun_out/r02/prof_cfg2_update.log
