# Update timing at configs 3, 2, 4 (current build vs var/head.so) + GPU suite + per-kernel launch list at config 3.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_upd_tests.log 2>&1; echo rc=$? >> gpurun_out/ab_upd_tests.log
L=paper_2603_09229_b200/_lib
for r in 1 2; do
  echo "head:"; FK_LIB_PATH=$L/var/head.so SHAPE=4,0,1 python scripts/update_small.py
  echo "new:"; SHAPE=4,0,1 python scripts/update_small.py
done > gpurun_out/ab_upd.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_hist|k_scan|k_scatter|k_segsum' --csv --log-file gpurun_out/ab_upd_launches.csv env SHAPE=4,0,1 python scripts/update_small.py > /dev/null 2>&1
