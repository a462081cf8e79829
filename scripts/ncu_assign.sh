#!/bin/bash
# usage: ncu_assign.sh <tag> [kernel-regex]
tag=$1; k=${2:-fk_assign_tc}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -f -o gpurun_out/prof_$tag python scripts/prof_assign.py > gpurun_out/prof_$tag.log 2>&1
tail -3 gpurun_out/prof_$tag.log
