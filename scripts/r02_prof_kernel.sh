#!/bin/bash
# ncu --set full of one kernel (regex $1) in scripts/update_small.py shapes ($2, comma list).
cd "$(dirname "$0")/.."
OUT=gpurun_out/r02
mkdir -p $OUT
for sh in ${2//,/ }; do
SHAPE=$sh timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s 3 -c 1 \
  -o $OUT/prof_${1}_shape$sh -f python scripts/update_small.py > /dev/null 2>&1; echo "ncu $1 shape $sh rc=$?"
done
