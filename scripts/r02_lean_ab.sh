#!/bin/bash
# A/B: lean role-warp paths (trace points and bound-analysis modes compiled out, slot counters
# instead of per-tile divisions) vs the build with runtime trace checks
# (paper_2603_09229_b200/_lib/ab/libfk_withtrace.so via FK_LIB_PATH); tests first.
cd "$(dirname "$0")/.."
python -m pytest -q -x tests/test_gpu_kernels.py tests/test_gpu_split.py tests/test_gpu_api.py tests/test_gpu_edges.py 2>&1 | tail -1
OLD=${OLD:-paper_2603_09229_b200/_lib/ab/libfk_withtrace.so}
for i in 1 2; do
  for lib in new old; do
    if [ $lib = old ]; then export FK_LIB_PATH=$OLD; else unset FK_LIB_PATH; fi
    echo "== $lib"
    python scripts/assign_time.py 64 16384 256 64 float16 50 2>&1 | tail -1
    python scripts/assign_time.py 1 1048576 1024 128 bfloat16 20 2>&1 | tail -1
    python scripts/assign_time.py 1 8388608 4096 128 bfloat16 5 2>&1 | tail -1
    python scripts/assign_time.py 1 1048576 1024 128 float32 5 2>&1 | tail -1
  done
done
unset FK_LIB_PATH
python scripts/config_perf.py 2>&1 | tail -4
