#!/bin/bash
# Round-2 ncu evidence of the bench command (one GPU): the launch list (per-launch times,
# cold-cache and serialized) and one --set full capture of FlashAssign and of each update kernel.
cd "$(dirname "$0")/.."
OUT=gpurun_out/r02
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > $OUT/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fk_assign_tc2 -s 1 -c 1 \
    -o $OUT/prof_assign -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $OUT/prof_assign.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_hist|k_colscan|k_scatter|k_segsum" -s 3 -c 3 \
    -o $OUT/prof_update -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $OUT/prof_update.log 2>&1
ls -la $OUT | tail -5
