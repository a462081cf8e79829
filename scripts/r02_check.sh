#!/bin/bash
# Round-2 GPU check: GPU tests, one bench line, the 2-rank rehearsal on one GPU.
cd "$(dirname "$0")/.."
OUT=gpurun_out/r02
mkdir -p $OUT
python -c "import torch; print(torch.cuda.get_device_name(0))"
timeout 1500 python -m pytest ${PYTEST_FILES:-tests} -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 $OUT/pytest_gpu.log
if [ -z "${SKIP_BENCH:-}" ]; then
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
tail -c 3000 $OUT/bench.json
FK_BENCH_SHARE_GPU=1 FK_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu \
  > $OUT/bench_share2.json 2> $OUT/bench_share2.err; echo "share2 rc=$?"
tail -c 1500 $OUT/bench_share2.json; tail -5 $OUT/bench_share2.err
timeout 120 python bench.py --gpus 2 --steps 2 --warmup 3 > $OUT/bench_gpus2_on_1.out 2>&1; echo "gpus2-on-1gpu rc=$? (must fail)"
tail -3 $OUT/bench_gpus2_on_1.out
fi
