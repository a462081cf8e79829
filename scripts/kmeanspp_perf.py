"""Device k-means++ seeding cost at scale (one GPU).

    python scripts/kmeanspp_perf.py [N] [d] [K] [dtype]

Reports ms per D^2 draw (sweep + pairwise total + certified select) and the
serial-fallback cost (FK_PP_FORCE_EXACT=1 in a second run), plus the oracle's
CPU time per draw on a sample for scale.
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_09229_b200 import ops  # noqa: E402
from paper_2603_09229_b200.core import kmeanspp_indices_device  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 23
d = int(sys.argv[2]) if len(sys.argv) > 2 else 128
K = int(sys.argv[3]) if len(sys.argv) > 3 else 256
dt = getattr(torch, sys.argv[4]) if len(sys.argv) > 4 else torch.bfloat16
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
centers = torch.rand(4096, d, device=dev, generator=g) * 20 - 10
lab = torch.randint(0, 4096, (N,), device=dev, generator=g)
x = (centers[lab] + torch.randn(N, d, device=dev, generator=g)).to(dt)[None].contiguous()
del centers, lab
first = torch.zeros(1, dtype=torch.int64, device=dev)
u = torch.rand(1, K - 1, dtype=torch.float64, device=dev, generator=g)
kw = min(K, 8)
ops.kmeanspp(x, kw, first, u[:, :kw - 1].contiguous())  # warm
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
idx, halted = ops.kmeanspp(x, K, first, u)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
bytes_per_draw = N * d * x.element_size() + 2 * N * 8
print(f"N={N} d={d} K={K} {dt}: {ms:.1f} ms total, {ms / (K - 1):.3f} ms/draw, "
      f"sweep-equivalent {bytes_per_draw / (ms / (K - 1)) / 1e6:.0f} GB/s (X + table r/w)")
t = time.time()
idx2 = kmeanspp_indices_device(x, K, 0)
print(f"public kmeanspp_indices_device (incl. host RNG + D2H): {(time.time() - t) * 1e3:.1f} ms")
