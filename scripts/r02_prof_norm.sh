#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
for c in 4 2; do
timeout 600 ncu --profile-from-start off -k regex:k_normalize -c 1 --set full --import-source on --clock-control none \
  -o gpurun_out/r02/prof_norm_cfg$c -f python scripts/iter_launches.py $c 1 > gpurun_out/r02/prof_norm_cfg$c.log 2>&1
tail -1 gpurun_out/r02/prof_norm_cfg$c.log
done
