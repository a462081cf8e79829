#!/bin/bash
# A/B: rolling-pair TMEM loads (FK_ASSIGN_EPI2=2) vs the default chunk schedule, config 3 assign
# (trace + timing) and the per-config table.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
python -m pytest -q -x tests/test_gpu_kernels.py -k "tc_assign" 2>&1 | tail -1
FK_ASSIGN_EPI2=2 python -m pytest -q -x tests/test_gpu_kernels.py -k "tc_assign or precomputed" 2>&1 | tail -1
for e in 2 d 2 d; do
  if [ $e = d ]; then unset FK_ASSIGN_EPI2; else export FK_ASSIGN_EPI2=$e; fi
  echo "== FK_ASSIGN_EPI2=${FK_ASSIGN_EPI2:-default}"
  python scripts/assign_time.py 1 8388608 4096 128 bfloat16 10 2>&1 | tail -1
  python scripts/assign_time.py 1 1048576 1024 128 bfloat16 20 2>&1 | tail -1
done
unset FK_ASSIGN_EPI2
FK_ASSIGN_EPI2=2 python scripts/trace_cfg3.py > /dev/null 2>&1; python scripts/trace_assign.py gpurun_out/r02/trace_cfg3_plain.txt | tail -5
