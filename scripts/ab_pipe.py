"""Same-box A/B of the Lloyd loop: iterate/poll/commit vs LloydEngine.run (speculative next assign)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2603_09229_b200 import LloydEngine
B, N, K, d = [int(v) for v in sys.argv[1:5]]
dt = getattr(torch, sys.argv[5]) if len(sys.argv) > 5 else torch.bfloat16
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 5
g = torch.Generator(device="cuda").manual_seed(0)
centers = torch.rand((B, K, d), device="cuda", generator=g) * 20 - 10
lab = torch.randint(0, K, (B, N), device="cuda", generator=g)
x = (torch.gather(centers, 1, lab[..., None].expand(B, N, d)) + torch.randn((B, N, d), device="cuda", generator=g)).to(dt).contiguous()
del centers, lab
c0 = torch.stack([x[b, torch.randperm(N, device="cuda", generator=g)[:K]] for b in range(B)]).float()
eng = LloydEngine(x, K)
eng.set_centroids(c0)
ev = lambda: torch.cuda.Event(enable_timing=True)
def old():
    for _ in range(reps):
        eng.iterate(); eng.poll(); eng.commit()
def pipe():
    eng.run(reps, -1.0, stop_on_repeat=False)
for f in (old, pipe, old, pipe):
    f()
torch.cuda.synchronize()
for r in range(3):
    for name, f in (("old", old), ("pipe", pipe)):
        torch.cuda.synchronize()
        a, b = ev(), ev(); a.record(); f(); b.record(); torch.cuda.synchronize()
        print(f"B={B} N={N} K={K}: {name:4s} {a.elapsed_time(b) / reps * 1e3:.1f} us/iter", flush=True)
