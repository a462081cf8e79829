"""Hot SASS instructions (stall samples) and the top stall reasons of one ncu report.
usage: python scripts/ncu_hot.py report.ncu-rep [top] [kernel-regex]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kf = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
raw = subprocess.run(["ncu", "-i", rep, *kf, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, v = r[0], r[2]
keys = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "smsp__inst_executed.sum"]
for k in keys:
    if k in h:
        print(f"{k:60s} {v[h.index(k)]}")
st = [(float(v[i]), h[i]) for i in range(len(h))
      if "average_warps_issue_stalled" in h[i] and h[i].endswith("per_issue_active.ratio") and v[i]]
for x in sorted(st, reverse=True)[:8]:
    print(f"  stall {x[1].split('stalled_')[1].split('_per')[0]:24s} {x[0]:.2f}")
src = subprocess.run(["ncu", "-i", rep, *kf, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
i = hh.index("Warp Stall Sampling (All Samples)")
ie = hh.index("Instructions Executed")
data = [(float(x[i] or 0), x[0], x[1].strip(), x[ie]) for x in rows[2:] if len(x) > i]
tot = sum(d[0] for d in data) or 1
print(f"SASS instructions {len(data)}, samples {tot:.0f}")
for n, d in enumerate(data):
    if d[0] / tot >= 0.01 or n in []:
        print(f"{n:5d} {d[0]/tot*100:5.1f}% {d[2][:80]:80s} ex={d[3]}")
