#!/bin/bash
# config-3 (and 2, 4) update: warp-table budget and the radix scatter (A/B)
cd "$(dirname "$0")/.."
for v in "FK_SW_TABLE_KB=64" "FK_SW_TABLE_KB=96" "FK_SW_TABLE_KB=160"; do
  echo "== $v"; env $v timeout 300 python scripts/config_perf.py 2>&1 | grep -E "cfg2|cfg3|cfg4 B"
done
