"""compute-sanitizer driver for the kernels added in round 2's second session (dev aid):
the assign epilogue's histogram fold and precomputed row norms (both epilogue layouts),
fk_update_prehist (scatter clearing sums/arrivals, segsum clearing the table), the
segment-chained k_segsum2, numpy-order objective partials (full and ragged buffers), and
the end-of-iteration launch in both forms (FK_TAIL is read once per process: fused here,
the split form through the three launches it would issue)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_09229_b200 import LloydEngine, ops  # noqa: E402

torch.manual_seed(0)
for (B, N, K, d, dt) in [(3, 5000, 200, 64, torch.float16), (1, 20000, 700, 128, torch.bfloat16),
                         (2, 3001, 37, 32, torch.bfloat16)]:
    x = (torch.randn(B, N, d, device="cuda") * 2).to(dt)
    c = x[:, :K].contiguous()
    fold = ops.hist_fold(x, K)
    xn = ops.assign_row_norms(x, K)
    for _ in range(2):
        ids, m = ops.assign(x, c, hist=fold, xnorm=xn)
        s, n = ops.update(x, ids, K, 777, hist=fold)
    ids2, m2 = ops.assign(x, c)
    s2, n2 = ops.update(x, ids2, K, 777)
    torch.cuda.synchronize()
    assert torch.equal(ids, ids2) and torch.equal(n, n2)
    assert torch.equal(s.view(torch.int64), s2.view(torch.int64))
for n in (1, 8191, 8192, 20001):
    mm = torch.rand(3, n, device="cuda")
    ops.objective(mm)
    part = torch.empty((3 * -(-n // ops.OBJ_BLOCK),), dtype=torch.float64, device="cuda")
    ops.objective_partials(mm, part)
x = (torch.randn(4, 3000, 64, device="cuda") * 3).half()
eng = LloydEngine(x, 64)
eng.set_centroids(x[:, :64].float())
eng.run(3, -1.0, stop_on_repeat=False)
eng.run(10, 1e30)
torch.cuda.synchronize()
print("ok")
