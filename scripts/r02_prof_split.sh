#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
for k in ${KLIST:-k_certify k_fallback_rows}; do
timeout 600 ncu --profile-from-start off -k regex:$k -c 1 --set full --import-source on --clock-control none \
  -o gpurun_out/r02/prof_$k -f python scripts/split_one.py gauss > gpurun_out/r02/prof_$k.log 2>&1
tail -3 gpurun_out/r02/prof_$k.log
done
