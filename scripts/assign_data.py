"""Assign-kernel time vs input distribution (dev aid)."""
import os, sys, torch
sys.path.insert(0, ".")
from paper_2603_09229_b200 import ops
N, K, d = 1 << 23, 4096, 128
torch.manual_seed(0)
def timeit(x, c):
    ids, mind = ops.assign(x, c)
    for _ in range(3): ops.assign(x, c, idx_out=ids, mind_out=mind)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(5): ops.assign(x, c, idx_out=ids, mind_out=mind)
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / 5
g = torch.Generator(device="cuda").manual_seed(0)
base = torch.randn(1, N, d, device="cuda", generator=g)
off = torch.randint(-10, 10, (1, 1, d), device="cuda", generator=g).float()
centers = torch.rand((K, d), device="cuda", generator=g) * 20 - 10
lab = torch.randint(0, K, (N,), device="cuda", generator=g)
cases = {
  "randn": base,
  "randn+offset": base + off,
  "blobs": (centers[lab] + base[0])[None],
  "zeros": torch.zeros_like(base),
}
for name, xf in cases.items():
    x = xf.to(torch.bfloat16).contiguous()
    for cname, c in [("first K", x[:, :K].contiguous()), ("random K", x[:, torch.randperm(N, device="cuda")[:K]].contiguous())]:
        t = timeit(x, c)
        print(f"{name:14s} {cname:9s} {t:7.3f} ms  {2*N*K*d/t/1e9:6.0f} TF/s")
