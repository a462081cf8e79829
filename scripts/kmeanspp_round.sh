mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kmeanspp.py -m gpu -x -q > gpurun_out/kpp_tests.log 2>&1; echo rc=$? >> gpurun_out/kpp_tests.log
for r in 1 2; do
  timeout 600 python scripts/kmeanspp_perf.py 8388608 128 512 bfloat16
  FK_PP_SWEEP=row1 timeout 600 python scripts/kmeanspp_perf.py 8388608 128 512 bfloat16
done > gpurun_out/kpp_perf.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_pp -c 20 --csv --log-file gpurun_out/kpp_launches.csv python scripts/kmeanspp_perf.py 8388608 128 4 bfloat16 > /dev/null 2>&1
