mkdir -p gpurun_out
for shape in "1 8388608 4096 128 bfloat16" "64 16384 256 64 float16" "1 1048576 1024 128 bfloat16"; do
  for m in 0; do
    FK_ASSIGN_DEBUG_MODE=$m python scripts/trace_cfg.py $shape gpurun_out/trace.txt
    echo "== mode $m $shape"; python scripts/trace_assign.py gpurun_out/trace.txt
  done
done > gpurun_out/trace_round.txt 2>&1
