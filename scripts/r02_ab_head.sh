#!/bin/bash
# Same-box A/B of two library builds on the bench command (FK_LIB_PATH=abl/libold.so vs the in-tree build).
cd "$(dirname "$0")/.."
for r in 1 2 3; do
  for v in old new; do
    if [ $v = old ]; then export FK_LIB_PATH=abl/libold.so; else unset FK_LIB_PATH; fi
    timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', round(d['ms_per_step'],3), 'assign', round(d['roofline']['ms_per_launch'],3), d['clocks']['reasons'])"
  done
done
