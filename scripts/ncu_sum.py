"""Summarize an ncu report: key throughput metrics + stall reasons (dev aid)."""
import csv, subprocess, sys, io
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "gpc__cycles_elapsed.max", "launch__grid_size"]
for r in rows[2:]:
    print("---")
    for k in want:
        if k in h:
            i = h.index(k); print(f"  {k} [{u[i]}] {r[i][:80]}")
    st = [(float(r[i]), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
          for i, k in enumerate(h) if k.startswith("smsp__average_warps_issue_stalled_") and r[i] not in ("", "n/a")]
    st.sort(reverse=True)
    print("  stalls:", ", ".join(f"{n}={v:.2f}" for v, n in st[:8]))
