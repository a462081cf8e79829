# A/B two library builds on the same box: bash scripts/ab_assign.sh libA.so libB.so [rounds]
for r in $(seq 1 ${3:-2}); do
  for lib in "$1" "$2"; do
    echo -n "$(basename $lib): "; FK_LIB_PATH=$lib MODES="0" bash scripts/assign_modes.sh | tail -1
  done
done
