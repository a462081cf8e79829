#!/bin/bash
# Config 4 FlashAssign: deeper X prefetch (8 slots for one K atom) and, with precomputed row norms,
# the X slot released by the MMA alone.  Tests, then plain / engine-style (hist + xnorm) timings and traces.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
python -m pytest -q -x tests/test_gpu_kernels.py -k "tc_assign or precomputed or hist_fold" 2>&1 | tail -1
python -m pytest -q -x tests/test_gpu_api.py tests/test_gpu_split.py 2>&1 | tail -1
for i in 1 2; do
  python scripts/assign_time.py 64 16384 256 64 float16 50 2>&1 | tail -1
  python scripts/assign_time.py 1 1048576 1024 128 bfloat16 20 2>&1 | tail -1
done
FK_ASSIGN_DEBUG_MODE=3 python scripts/trace_cfg3.py 64 16384 256 64 > /dev/null 2>&1
python scripts/trace_assign.py gpurun_out/r02/trace_cfg3_plain.txt | tail -5
python scripts/trace_assign.py gpurun_out/r02/trace_cfg3_fold_xnorm.txt | tail -5
python scripts/trace_xload.py gpurun_out/r02/trace_cfg3_fold_xnorm.txt | tail -6
python scripts/config_perf.py 2>&1 | tail -4
