# k-means++ device seeding: scale timing + kernel profile (one GPU)
mkdir -p gpurun_out
timeout 300 python scripts/kmeanspp_perf.py 8388608 128 128 bfloat16 > gpurun_out/kpp_perf.log 2>&1
FK_PP_SWEEP=tile timeout 300 python scripts/kmeanspp_perf.py 8388608 128 128 bfloat16 >> gpurun_out/kpp_perf.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_pp -c 40 --csv --log-file gpurun_out/kpp_launches.csv python scripts/kmeanspp_perf.py 8388608 128 4 bfloat16 > gpurun_out/kpp_ncu1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_pp_sweep -s 2 -c 1 -o gpurun_out/kpp_sweep_pipe -f python scripts/kmeanspp_perf.py 8388608 128 4 bfloat16 > gpurun_out/kpp_ncu2.log 2>&1
FK_PP_SWEEP=tile timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_pp_sweep -s 2 -c 1 -o gpurun_out/kpp_sweep_tile -f python scripts/kmeanspp_perf.py 8388608 128 4 bfloat16 > gpurun_out/kpp_ncu3.log 2>&1
