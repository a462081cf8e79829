#!/bin/bash
# fp8 bias step A/B: integer-grid parity, random-data differences vs the bf16 step, timings, ncu kernel times.
cd "$(dirname "$0")/.."
O=gpurun_out/r02b8; mkdir -p $O
FK_ASSIGN_BIAS8=1 timeout 300 python scripts/r02_bias8_ab.py --grid
for r in 1 2; do
  echo "== bf16 bias step"; FK_ASSIGN_BIAS8=0 timeout 300 python scripts/r02_bias8_ab.py $O/b16.npz
  echo "== fp8 bias step"; FK_ASSIGN_BIAS8=1 timeout 300 python scripts/r02_bias8_ab.py $O/b8.npz
done
python scripts/r02_bias8_ab.py --compare $O/b16.npz $O/b8.npz
for v in 0 1; do
  FK_ASSIGN_BIAS8=$v timeout 300 ncu --metrics gpu__time_duration.sum -k regex:fk_assign_tc2 --clock-control none \
    python scripts/assign_time.py 1 8388608 4096 128 bfloat16 3 2>&1 | grep -E "gpu__time_duration" | tail -3
done
