#!/bin/bash
# Multicast-quad FlashAssign A/B on one box: pair kernel vs quads (+ the pair kernel on the SMs
# the 4-CTA clusters cannot use), same shapes, bitwise hash check.
cd "$(dirname "$0")/.."
for r in 1 2; do
for cfg in "0 1" "1 1.12" "1 1.05" "1 1.2"; do
  set -- $cfg
  echo "== FK_ASSIGN_MC=$1 FK_ASSIGN_MC_GAIN=$2 (round $r)"
  FK_ASSIGN_MC=$1 FK_ASSIGN_MC_GAIN=$2 FK_ASSIGN_MC_VERBOSE=1 timeout 300 python scripts/r02_mc_ab.py 2>&1 | tail -8
done
done
