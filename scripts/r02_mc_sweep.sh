#!/bin/bash
# Quads + pair kernel: how many extra pairs co-run with the 33 quads (FK_ASSIGN_MC_EXTRA), configs 3 and 2.
cd "$(dirname "$0")/.."
for r in 1 2; do
  echo "== pair kernel only"; FK_ASSIGN_MC=0 SHAPES=0,1 timeout 300 python scripts/r02_mc_ab.py 2>&1 | tail -2
  for ex in 0 2 4 6 8; do
    for g in 1.12; do
      echo "== quads + $ex pairs, gain $g"
      FK_ASSIGN_MC=1 FK_ASSIGN_MC_EXTRA=$ex FK_ASSIGN_MC_GAIN=$g SHAPES=0,1 timeout 300 python scripts/r02_mc_ab.py 2>&1 | tail -2
    done
  done
done
