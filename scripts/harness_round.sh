# Reference-schema bench sweep, time-to-first-run and tile search on one GPU.
mkdir -p gpurun_out
M="python -m paper_2603_09229_b200.benchmark"
timeout 600 $M bench --n 1048576 --k 1024 --d 128 --dtype bf16 --reps 5 --out gpurun_out/bench_sweep_cfg2.csv
timeout 600 $M bench --n 16384 --k 256 --d 64 --b 64 --dtype fp16 --reps 5 --out gpurun_out/bench_sweep_cfg4.csv
timeout 600 $M bench --n 65536 --k 1024 --d 128 --dtype single --reps 5 --out gpurun_out/bench_sweep_f32.csv
timeout 600 $M ttfr --shapes 1048576:1024:128:1,8388608:4096:128:1,8388608:65536:128:1,16384:256:64:64,100000:777:96:3 --out gpurun_out/ttfr.csv
timeout 900 $M tune --n 1048576 --k 1024 --d 128 --dtype bf16 --reps 3 --out gpurun_out/tune_cfg2.csv
