#!/bin/bash
# time-to-first-run per new shape (kernels preloaded at device bind)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
timeout 600 python -m paper_2603_09229_b200.benchmark ttfr --shapes 1048576:1024:128:1,16384:256:64:64,100000:777:96:3,65536:1024:128:1 --out gpurun_out/r02/ttfr.csv
timeout 600 python -m paper_2603_09229_b200.benchmark ttfr --dtype single --shapes 65536:1024:128:1,10000:8:16:1 --out gpurun_out/r02/ttfr_f32.csv
