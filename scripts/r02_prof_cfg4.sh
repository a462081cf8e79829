#!/bin/bash
# ncu --set full of one config-4 FlashAssign launch (fused path unless FK_ASSIGN_FUSE=0)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
timeout 600 ncu --profile-from-start off -k regex:fk_assign_tc2 -c 1 --set full --import-source on --clock-control none \
  -o gpurun_out/r02/prof_fused_cfg4 -f python scripts/iter_launches.py 4 1 > gpurun_out/r02/prof_fused_cfg4.log 2>&1
tail -1 gpurun_out/r02/prof_fused_cfg4.log
