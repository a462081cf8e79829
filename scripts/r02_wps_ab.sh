#!/bin/bash
# segsum warp slices per SM (A/B, interleaved), configs 2/3/4
cd "$(dirname "$0")/.."
for v in 32 16 24 48 32 16; do echo "== FK_SEGSUM_WPS=$v"; FK_SEGSUM_WPS=$v timeout 300 python scripts/config_perf.py 2>&1 | grep -E "cfg2|cfg3|cfg4 B" | sed 's/.*\(cfg[0-9]\).*update \([0-9.]* us\).*/\1 update \2/'; done
