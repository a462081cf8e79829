#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
for tool in memcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_r02b.py > gpurun_out/r02/sanitizer_r02b_$tool.txt 2>&1
  echo "== $tool rc=$?"; tail -4 gpurun_out/r02/sanitizer_r02b_$tool.txt
done
