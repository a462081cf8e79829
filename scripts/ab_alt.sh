mkdir -p gpurun_out
for r in 1 2; do for a in 1 0; do for e in 0 1; do
  echo "alt=$a epi2=$e: $(FK_ASSIGN_ALT=$a FK_ASSIGN_EPI2=$e python scripts/trace_cfg.py 64 16384 256 64 float16 /tmp/t.txt | tail -1)"
done; done; done > gpurun_out/ab_alt.txt 2>&1
FK_ASSIGN_ALT=0 timeout 300 python -m pytest tests/test_gpu_edges.py tests/test_gpu_kernels.py -m gpu -x -q >> gpurun_out/ab_alt.txt 2>&1
