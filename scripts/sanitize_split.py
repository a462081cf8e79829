"""compute-sanitizer driver for the round-2 kernels (dev aid): the certified f32/f64
split path (both epilogue layouts, candidates, full fallback with duplicated
centroids), the f64 serial segsum, the fused normalize + loop tail (engine), and
the device top-E."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_09229_b200 import LloydEngine, ops  # noqa: E402

torch.manual_seed(0)
for (B, N, K, d, dt) in [(1, 3000, 1000, 128, torch.float32), (2, 1500, 200, 64, torch.float64),
                         (1, 777, 300, 24, torch.float32)]:
    x = torch.randn(B, N, d, device="cuda", dtype=dt)
    c = x[:, :K].contiguous()
    c[:, K // 2:] = c[:, : K - K // 2]  # duplicated centroids: candidates / fallback rows
    ids, mind = ops.assign(x, c, path="split")
    ids2, mind2 = ops.assign(x, c, path="mirror")
    torch.cuda.synchronize()
    assert torch.equal(ids, ids2) and torch.equal(mind, mind2)
    s, n = ops.update(x.double(), ids, K, 512)
torch.cuda.synchronize()
x = (torch.randn(4, 3000, 64, device="cuda") * 3).half()
eng = LloydEngine(x, 64)
eng.set_centroids(x[:, :64].float())
eng.run(3, -1.0, stop_on_repeat=False)
m = torch.rand(2, 50000, device="cuda")
idx = ops.farthest(m, 100) if hasattr(ops, "farthest") else None
torch.cuda.synchronize()
print("ok")
