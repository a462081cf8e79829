# k-means++ device seeding: parity tests, scale timing, kernel profile (one GPU)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kmeanspp.py -m gpu -x -q > gpurun_out/kpp_tests.log 2>&1; echo rc=$? >> gpurun_out/kpp_tests.log
timeout 300 python scripts/kmeanspp_perf.py 8388608 128 128 bfloat16 > gpurun_out/kpp_perf.log 2>&1
FK_PP_SWEEP=pipe timeout 300 python scripts/kmeanspp_perf.py 8388608 128 128 bfloat16 >> gpurun_out/kpp_perf.log 2>&1
timeout 300 python scripts/kmeanspp_perf.py 8388608 128 64 float32 >> gpurun_out/kpp_perf.log 2>&1
timeout 300 python scripts/kmeanspp_perf.py 16384 64 256 float16 >> gpurun_out/kpp_perf.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_pp -c 40 --csv --log-file gpurun_out/kpp_launches.csv python scripts/kmeanspp_perf.py 8388608 128 4 bfloat16 > gpurun_out/kpp_ncu1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_pp_sweep -s 2 -c 1 -o gpurun_out/kpp_sweep_tile -f python scripts/kmeanspp_perf.py 8388608 128 4 bfloat16 > gpurun_out/kpp_ncu3.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2603_09229_b200/csrc scripts/probe_tmem_ld.cu -o /tmp/probe_ld && timeout 120 /tmp/probe_ld > gpurun_out/probe_tmem_ld.txt 2>&1
