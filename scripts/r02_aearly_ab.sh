#!/bin/bash
# A/B: X slot released right after the row tile's last data MMA (FK_ASSIGN_AEARLY=1, default)
# vs after the bias step and the accumulator commit (0): tests, config 4/2/3 assign, traces.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
python -m pytest -q -x tests/test_gpu_kernels.py -k "tc_assign or precomputed or hist_fold" 2>&1 | tail -1
python -m pytest -q -x tests/test_gpu_split.py 2>&1 | tail -1
for e in 1 0 1 0; do
  echo "== FK_ASSIGN_AEARLY=$e"
  FK_ASSIGN_AEARLY=$e python scripts/assign_time.py 64 16384 256 64 float16 50 2>&1 | tail -1
  FK_ASSIGN_AEARLY=$e python scripts/assign_time.py 1 1048576 1024 128 bfloat16 20 2>&1 | tail -1
  FK_ASSIGN_AEARLY=$e python scripts/assign_time.py 1 8388608 4096 128 bfloat16 5 2>&1 | tail -1
done
for e in 1 0; do
  echo "== trace cfg4 FK_ASSIGN_AEARLY=$e"
  FK_ASSIGN_AEARLY=$e python scripts/trace_cfg3.py 64 16384 256 64 > /dev/null 2>&1
  python scripts/trace_assign.py gpurun_out/r02/trace_cfg3_plain.txt | tail -5
done
