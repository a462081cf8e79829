#!/bin/bash
# A/B: fewest points per update block (FK_UPDATE_MINPTS) -- more scatter blocks for small N.
cd "$(dirname "$0")/.."
for v in 8192 4096 2048 8192 4096 2048; do
  echo "== FK_UPDATE_MINPTS=$v"
  FK_UPDATE_MINPTS=$v timeout 300 python scripts/config_perf.py 2>&1 | tail -4
done
