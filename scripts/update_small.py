"""ops.update at configs 2, 4 and 3 under a CUDA graph (for A/B and ncu launch lists; dev aid).
    FK_UPDATE_CLUSTER=0 selects the global sort path for the small shapes."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2603_09229_b200 import ops
shapes = [(1, 1 << 20, 1024, 128, torch.bfloat16), (64, 16384, 256, 64, torch.float16),
          (64, 16384, 256, 64, torch.bfloat16), (8, 65536, 256, 64, torch.bfloat16),
          (1, 1 << 23, 4096, 128, torch.bfloat16)]
import os
if os.environ.get("SHAPE"):
    shapes = [shapes[int(v)] for v in os.environ["SHAPE"].split(",")]
for (B, N, K, d, dt) in shapes:
    x = torch.randn(B, N, d, device="cuda").to(dt)
    ids = torch.randint(0, K, (B, N), device="cuda", dtype=torch.int32)
    sums = torch.empty((B, K, d), dtype=torch.float64, device="cuda")
    counts = torch.empty((B, K), dtype=torch.int64, device="cuda")
    m = torch.zeros((), dtype=torch.int64, device="cuda")
    for _ in range(3):
        ops.update(x, ids, K, 16384, sums=sums, counts=counts, merges=m)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ops.update(x, ids, K, 16384, sums=sums, counts=counts, merges=m)
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(20): g.replay()
    e.record(); e.synchronize()
    t = s.elapsed_time(e) / 20 * 1e3
    by = B * N * d * x.element_size() + 4 * B * N + 4 * B * K * d + 4 * B * K
    print(f"B={B} N={N} K={K} d={d} {dt}: {t:.1f} us  {by / t / 1e3:.0f} GB/s")
