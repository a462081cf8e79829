# Per-kernel launch list of the update at configs 2 and 4 + config perf.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_hist|k_scan|k_scatter|k_segsum' --csv --log-file gpurun_out/upd24_launches.csv env SHAPE=0,1 python scripts/update_small.py > /dev/null 2>&1
timeout 400 python scripts/config_perf.py > gpurun_out/config_perf.txt 2>&1
