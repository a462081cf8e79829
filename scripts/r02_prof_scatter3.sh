#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
timeout 600 ncu --profile-from-start off -k regex:${KREGEX:-k_scatter_warp} -c 1 --set full --import-source on --clock-control none \
  -o gpurun_out/r02/prof_${KREGEX:-k_scatter_warp}_cfg3 -f python scripts/iter_launches.py 3 1 > gpurun_out/r02/prof_scatter_cfg3.log 2>&1
tail -1 gpurun_out/r02/prof_scatter_cfg3.log
