# A/B the ||c||^2 bias placements of the FlashAssign pair kernel on one box
# (FK_ASSIGN_BIAS: 0 epilogue, 1 bias-in-GEMM, 2 TMEM seed).
mkdir -p gpurun_out
FK_ASSIGN_BIAS=2 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_edges.py -m gpu -x -q > gpurun_out/ab_bias_tests_2.log 2>&1; echo rc=$? >> gpurun_out/ab_bias_tests_2.log
for r in 1 2; do
  for b in 1 2; do
    echo -n "bias=$b: "; FK_ASSIGN_BIAS=$b MODES=0 bash scripts/assign_modes.sh | tail -1
  done
done > gpurun_out/ab_bias.txt 2>&1
