#!/bin/bash
# FlashAssign epilogue variants (same box, interleaved): default vs chunk pairs everywhere
cd "$(dirname "$0")/.."
for v in "X=0" "FK_ASSIGN_EPI2=1" "X=0" "FK_ASSIGN_EPI2=1"; do echo "== $v"; env $v timeout 300 python scripts/config_perf.py 2>&1 | grep -E "cfg2|cfg3|cfg4 B" | sed 's/| update.*//'; done
