"""Print the in-kernel pipeline timeline written by FK_ASSIGN_TRACE (dev aid)."""
import sys
rows = [list(map(int, l.split())) for l in open(sys.argv[1]) if l.strip()]
names = ["mma_start", "mma_issued", "epi_tfull", "epi_release", "epi_done", "prod_issued", "mma_wait_empty", "mma_a_full"]
t0 = rows[0][0]
print("g   " + " ".join(f"{n:>13s}" for n in names))
prev = None
for g, r in enumerate(rows):
    print(f"{g:3d} " + " ".join(f"{(v - t0) if v else -1:13d}" for v in r[:8]))
d = [rows[i + 1][0] - rows[i][0] for i in range(len(rows) - 1)]
print("mean MMA period (cycles):", sum(d) / len(d))
ep = [r[4] - r[2] for r in rows]
print("mean epilogue busy per tile:", sum(ep) / len(ep))
wait = [r[0] - r[6] for r in rows]
print("mean MMA wait on t_empty:", sum(wait) / len(wait))
lat = [r[2] - r[1] for r in rows]
print("mean issue->epi t_full seen:", sum(lat) / len(lat))
aw = [rows[i + 1][7] - rows[i][1] for i in range(len(rows) - 1) if rows[i + 1][7]]
if aw:
    print("mean MMA stall on a_full (row-tile starts):", sum(aw) / len(aw), "over", len(aw))
