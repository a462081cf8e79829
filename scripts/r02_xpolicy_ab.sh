#!/bin/bash
# FlashAssign X-load L2 policy / tensor-map L2 promotion A/B (library variants built by scripts/build_variant.sh).
cd "$(dirname "$0")/.."
for r in 1 2; do
  for lib in default abl/lib_xnormal.so abl/lib_promo_none.so abl/lib_promo128.so; do
    if [ $lib = default ]; then unset FK_LIB_PATH; else export FK_LIB_PATH=$lib; fi
    echo "== $lib"
    timeout 120 python scripts/assign_time.py 64 16384 256 64 float16 200
    timeout 120 python scripts/assign_time.py 1 1048576 1024 128 bfloat16 200
    timeout 120 python scripts/assign_time.py 1 8388608 4096 128 bfloat16 20
  done
done
