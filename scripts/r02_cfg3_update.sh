#!/bin/bash
# Config-3 update kernels on bench-like data (blob assignments): launch list, default and radix scatter.
cd "$(dirname "$0")/.."
OUT=gpurun_out/r02
mkdir -p $OUT
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/iter_launches_cfg3.csv python scripts/iter_launches.py 3 2 > /dev/null 2>&1
echo "== config 3 launches (2 iterations)"; python scripts/launch_table.py $OUT/iter_launches_cfg3.csv
python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2603_09229_b200 import LloydEngine, ops
B, N, K, d = 1, 1 << 23, 4096, 128
g = torch.Generator(device="cuda").manual_seed(0)
centers = torch.rand((B, K, d), device="cuda", generator=g) * 20 - 10
lab = torch.randint(0, K, (B, N), device="cuda", generator=g)
x = (torch.gather(centers, 1, lab[..., None].expand(B, N, d)) + torch.randn((B, N, d), device="cuda", generator=g)).to(torch.bfloat16)
c0 = torch.stack([x[b, torch.randperm(N, device="cuda", generator=g)[:K]] for b in range(B)]).float()
ids, _ = ops.assign(x, c0.to(torch.bfloat16))
cnt = torch.bincount(ids[0].long(), minlength=K)
print("cluster sizes: min", int(cnt.min()), "max", int(cnt.max()), "mean", float(cnt.float().mean()))
ev = lambda: torch.cuda.Event(enable_timing=True)
for _ in range(3): ops.update(x, ids, K, N)
torch.cuda.synchronize(); a, b = ev(), ev(); a.record()
for _ in range(10): ops.update(x, ids, K, N)
b.record(); torch.cuda.synchronize(); print("update on blob ids: %.1f us" % (a.elapsed_time(b) / 10 * 1e3))
ids2 = torch.randint(0, K, (B, N), device="cuda", dtype=torch.int32)
for _ in range(3): ops.update(x, ids2, K, N)
torch.cuda.synchronize(); a.record()
for _ in range(10): ops.update(x, ids2, K, N)
b.record(); torch.cuda.synchronize(); print("update on uniform ids: %.1f us" % (a.elapsed_time(b) / 10 * 1e3))
PY
