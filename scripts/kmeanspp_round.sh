mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kmeanspp.py -m gpu -x -q > gpurun_out/kpp_tests.log 2>&1; echo rc=$? >> gpurun_out/kpp_tests.log
FK_PP_FORCE_EXACT=1 timeout 900 python -m pytest tests/test_gpu_kmeanspp.py tests/test_gpu_acceptance.py -m gpu -x -q -k "kmeanspp or reference or oracle" >> gpurun_out/kpp_tests.log 2>&1; echo rc_forced=$? >> gpurun_out/kpp_tests.log
{
FK_PP_FORCE_EXACT=1 timeout 300 python scripts/kmeanspp_perf.py 8388608 128 16 bfloat16
FK_PP_FORCE_EXACT=1 FK_PP_EXACT_SERIAL=1 timeout 300 python scripts/kmeanspp_perf.py 8388608 128 16 bfloat16
timeout 600 python scripts/kmeanspp_perf.py 8388608 128 1024 bfloat16
FK_PP_PRUNE=0 timeout 600 python scripts/kmeanspp_perf.py 8388608 128 1024 bfloat16
} > gpurun_out/kpp_perf.log 2>&1
