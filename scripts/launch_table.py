"""Summarize an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel, the
durations in launch order (us).  usage: python scripts/launch_table.py file.csv"""
import collections
import csv
import io
import sys

txt = open(sys.argv[1]).read().split("\n")
i = next(j for j, l in enumerate(txt) if l.startswith('"ID"'))
agg = collections.OrderedDict()
for r in csv.DictReader(io.StringIO("\n".join(txt[i:]))):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    k = r["Kernel Name"].split("(")[0] + " grid" + r["Grid Size"]
    agg.setdefault(k, []).append(float(r["Metric Value"]) / 1e3)
for k, v in agg.items():
    print(f"{k[:70]:70s} n={len(v):3d} med={sorted(v)[len(v)//2]:8.1f} us  " + " ".join(f"{x:.1f}" for x in v[:6]))
