#!/bin/bash
# Update / iteration timing at configs 2-4 plus an ncu launch list of the update kernels.
cd "$(dirname "$0")/.."
OUT=gpurun_out/r02
mkdir -p $OUT
timeout 300 python scripts/update_small.py 2>&1 | tee $OUT/update_small.txt
timeout 600 python scripts/config_perf.py 2>&1 | tee $OUT/config_perf.txt
SHAPE=0,1,4 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_hist|k_colscan|k_scan|k_scatter|k_segsum' \
  --csv --log-file $OUT/update_launches.csv python scripts/update_small.py > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.DictReader(open("gpurun_out/r02/update_launches.csv")))
agg = collections.OrderedDict()
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum": continue
    k = r["Kernel Name"].split("(")[0]
    agg.setdefault(k, []).append(float(r["Metric Value"]))
for k, v in agg.items():
    print(f"{k:50s} n={len(v):3d} " + " ".join(f"{x/1e3:.1f}" for x in v[:12]) + " us")
PY
