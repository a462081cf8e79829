mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/s1_gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s1_pytest.log 2>&1; echo rc=$? >> gpurun_out/s1_pytest.log
timeout 300 python bench.py > gpurun_out/s1_bench.json 2> gpurun_out/s1_bench.err
for r in 1 2; do for b in 0 1; do echo -n "bias=$b: "; FK_ASSIGN_BIAS=$b MODES="0 1" bash scripts/assign_modes.sh | tr '\n' ' '; echo; done; done > gpurun_out/s1_ab_bias.txt 2>&1
