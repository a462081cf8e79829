#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
timeout 900 python scripts/split_perf.py 2>&1 | tee gpurun_out/r02/split_perf.txt
FK_SPLIT_NOFALLBACK=1 timeout 900 python scripts/split_perf.py 2>&1 | sed 's/^/[nofallback] /' | tee -a gpurun_out/r02/split_perf.txt
timeout 600 python scripts/f64_update_perf.py 2>&1 | tee gpurun_out/r02/f64_update_perf.txt
FK_SEGSUM_F64=parallel timeout 600 python scripts/f64_update_perf.py 2>&1 | tee -a gpurun_out/r02/f64_update_perf.txt
