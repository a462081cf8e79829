"""Write profiles/ncu_summary.json (+ a text summary) from ncu reports (dev aid).

usage: python scripts/make_ncu_summary.py <tag> gpurun_out/prof_assign.ncu-rep gpurun_out/prof_update.ncu-rep
"""
import csv, io, json, os, subprocess, sys

tag = sys.argv[1]
out = {}
lines = []
for rep in sys.argv[2:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    def val(r, k):
        i = h.index(k)
        v = float(r[i])
        unit = u[i]
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}.get(unit, 1)
        return v * scale
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        key = next((k for k in ("fk_assign_tc2", "fk_assign_tc", "k_segsum", "k_scatter_warp", "k_scatter_staged",
                                "k_scatter_block", "k_hist", "k_colscan", "k_scan")
                    if k in name), name[:40])
        if key == "fk_assign_tc2":
            key = "fk_assign_tc"
        rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
        t = val(r, "gpu__time_duration.sum")
        rec = {"kernel": name[:120], "dram_bytes": rd + wr, "dram_read": rd, "dram_write": wr,
               "duration_s": t}
        for k in ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                  "dram__throughput.avg.pct_of_peak_sustained_elapsed",
                  "smsp__issue_active.avg.pct_of_peak_sustained_active",
                  "lts__throughput.avg.pct_of_peak_sustained_elapsed",
                  "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"):
            if k in h:
                rec[k] = float(r[h.index(k)] or 0)
        out[key] = rec
        lines.append(f"{key:16s} {t*1e3:8.3f} ms  DRAM {rd/1e9:7.3f} GB read {wr/1e6:8.2f} MB written  "
                     + "  ".join(f"{k.split('.')[0].split('__')[1]}={rec[k]:.1f}" for k in rec if k.endswith("active") or k.endswith("elapsed")))
os.makedirs("profiles", exist_ok=True)
json.dump({"round": tag, "source": "ncu --set full --clock-control none (scripts/r02_ncu.sh)", **out},
          open("profiles/ncu_summary.json", "w"), indent=1)
open(f"profiles/{tag}_ncu_full.txt", "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
