#!/bin/bash
# histogram/scatter blocks per SM (A/B), configs 2/3/4
cd "$(dirname "$0")/.."
for v in 2 3 4 6; do echo "== FK_UPDATE_BPS=$v"; FK_UPDATE_BPS=$v timeout 300 python scripts/config_perf.py 2>&1 | grep -E "cfg2|cfg3|cfg4 B"; done
