#!/bin/bash
# X-load L2 policy A/B at config 3: evict-first (default) vs evict-normal, 5 alternations, plus the bench.
cd "$(dirname "$0")/.."
for r in 1 2 3 4 5; do
  for lib in default abl/lib_xnormal.so; do
    if [ $lib = default ]; then unset FK_LIB_PATH; else export FK_LIB_PATH=$lib; fi
    echo "$lib $(timeout 120 python scripts/assign_time.py 1 8388608 4096 128 bfloat16 30)"
  done
done
for r in 1 2; do
  for lib in default abl/lib_xnormal.so; do
    if [ $lib = default ]; then unset FK_LIB_PATH; else export FK_LIB_PATH=$lib; fi
    timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('bench $lib', round(d['ms_per_step'],3), 'assign', round(d['roofline']['ms_per_launch'],3), d['clocks']['reasons'])"
  done
done
