# A/B: minimum points per hist/scatter block (FK_UPDATE_MIN_RANGE), configs 3, 2, 4 update.
mkdir -p gpurun_out
for r in 1 2; do
  for m in 2048 8192 16384 32768; do
    echo "min_range=$m:"; FK_UPDATE_MIN_RANGE=$m SHAPE=4,0,1 python scripts/update_small.py
  done
done > gpurun_out/ab_bpb.txt 2>&1
FK_UPDATE_MIN_RANGE=16384 timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k update > gpurun_out/ab_bpb_tests.log 2>&1; echo rc=$? >> gpurun_out/ab_bpb_tests.log
