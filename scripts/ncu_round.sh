#!/bin/bash
# ncu evidence for the hot-path kernels (run under gpurun, one GPU).
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fk_assign_tc2 -s 1 -c 1 \
    -o gpurun_out/prof_assign -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/prof_assign.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_hist|k_scan|k_scatter|k_segsum" -s 4 -c 4 \
    -o gpurun_out/prof_update -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/prof_update.log 2>&1
ls -la gpurun_out
