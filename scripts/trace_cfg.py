"""In-kernel FlashAssign timeline (FK_ASSIGN_TRACE) at a given shape (dev aid).
    python scripts/trace_cfg.py B N K d dtype out.txt"""
import os, sys, torch
sys.path.insert(0, ".")
from paper_2603_09229_b200 import ops
B, N, K, d = map(int, sys.argv[1:5])
dt = getattr(torch, sys.argv[5])
torch.manual_seed(0)
x = torch.randn(B, N, d, device="cuda").to(dt)
c = x[:, :K].contiguous()
ids, mind = ops.assign(x, c)
for _ in range(10): ops.assign(x, c, idx_out=ids, mind_out=mind)
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(10): ops.assign(x, c, idx_out=ids, mind_out=mind)
e.record(); torch.cuda.synchronize()
print(f"B={B} N={N} K={K} d={d}: {s.elapsed_time(e)/10*1e3:.1f} us per assign")
os.environ["FK_ASSIGN_TRACE"] = sys.argv[6]
ops.assign(x, c, idx_out=ids, mind_out=mind)
