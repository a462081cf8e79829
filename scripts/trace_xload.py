"""X row-tile load issue vs MMA a_full pass (FK_ASSIGN_DEBUG_MODE=3 trace; dev aid).
usage: python scripts/trace_xload.py trace.txt"""
import sys
rows = [list(map(int, l.split())) for l in open(sys.argv[1]) if l.strip()]
t0 = rows[0][0]
print("g   x_issued  mma_a_full  mma_start  mma_issued   (a_full - x_issued)")
for g, r in enumerate(rows):
    xi, af = r[5], r[7]
    print(f"{g:3d} {xi - t0 if xi else -1:9d} {af - t0 if af else -1:11d} {r[0] - t0:10d} {r[1] - t0:11d}   "
          f"{(af - xi) if (xi and af) else -1}")
