"""Time one FlashAssign shape (dev aid): python scripts/assign_time.py B N K d [dtype] [iters]."""
import sys, torch
sys.path.insert(0, ".")
from paper_2603_09229_b200 import ops
B, N, K, d = (int(v) for v in sys.argv[1:5])
dt = getattr(torch, sys.argv[5]) if len(sys.argv) > 5 else torch.bfloat16
it = int(sys.argv[6]) if len(sys.argv) > 6 else 10
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(B, N, d, device="cuda", generator=g).to(dt)
c = x[:, :K].contiguous()
ids, mind = ops.assign(x, c)
for _ in range(3):
    ops.assign(x, c, idx_out=ids, mind_out=mind)
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(it):
    ops.assign(x, c, idx_out=ids, mind_out=mind)
e.record()
torch.cuda.synchronize()
t = s.elapsed_time(e) / it
print(f"B={B} N={N} K={K} d={d}: {t:.3f} ms {2*B*N*K*d/t/1e9:.0f} TF/s")
