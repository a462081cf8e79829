#!/bin/bash
# ncu launch lists (gpu__time_duration, cold, serialized) of one pipelined Lloyd iteration at configs 2 and 4.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
for c in 2 4; do
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/r02/cfg${c}_launches.csv python scripts/iter_launches.py $c 2 \
    > gpurun_out/r02/cfg${c}_launches.log 2>&1
  echo "cfg$c rc=$?"
done
