"""Per-rank Lloyd iteration time for config 3 split over P ranks (one GPU; dev aid).

Times LloydEngine.run on N/P points (K=4096, d=128, bf16) -- the compute each
rank performs per iteration in the point-sharded run -- to project strong
scaling before 8 GPUs are available.  The NCCL all-reduce of the packed 4.2 MB
buffer is not included (measured separately when several GPUs are present)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2603_09229_b200 import LloydEngine

K, d, N = 4096, 128, 1 << 23
for P in (1, 2, 4, 8):
    n = N // P
    g = torch.Generator(device="cuda").manual_seed(0)
    centers = torch.rand((1, 4096, d), device="cuda", generator=g) * 20 - 10
    lab = torch.randint(0, 4096, (1, n), device="cuda", generator=g)
    x = (centers[0][lab] + torch.randn((1, n, d), device="cuda", generator=g)).to(torch.bfloat16)
    del centers, lab
    eng = LloydEngine(x, K)
    eng.set_centroids(x[:, :K].float())
    eng.run(4, -1.0, stop_on_repeat=False)
    eng.run(3, -1.0, stop_on_repeat=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    reps = 10
    a.record()
    its, _, _ = eng.run(reps, -1.0, stop_on_repeat=False)
    b.record(); torch.cuda.synchronize()
    t = a.elapsed_time(b) / its
    print(f"P={P}: {n} points per rank, {t:.3f} ms per iteration (compute only)", flush=True)
    del eng, x
    torch.cuda.empty_cache()
