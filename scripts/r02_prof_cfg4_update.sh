#!/bin/bash
# ncu --set full of the config-4 update + normalize-tail kernels (one iteration)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
FK_SEGSUM_SEQ=${FK_SEGSUM_SEQ:-1} timeout 600 ncu --profile-from-start off -k "regex:k_segsum|k_normalize|k_scatter_warp|k_hist" -c 4 --set full \
  --import-source on --clock-control none -o gpurun_out/r02/prof_cfg4_update -f python scripts/iter_launches.py 4 1 \
  > gpurun_out/r02/prof_cfg4_update.log 2>&1
tail -2 gpurun_out/r02/prof_cfg4_update.log
