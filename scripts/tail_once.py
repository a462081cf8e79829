"""A few eager fk_normalize_loop_tail launches at BASELINE config 4 (ncu target, dev aid)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_09229_b200 import LloydEngine, ops  # noqa: E402

B, N, K, d, dt = (64, 16384, 256, 64, torch.float16) if (len(sys.argv) < 2 or sys.argv[1] == "4") else \
    (1, 1 << 20, 1024, 128, torch.bfloat16)
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn((B, N, d), device="cuda", generator=g).to(dt)
e = LloydEngine(x, K)
e.set_centroids(x[:, :K].float())
e.iterate(); e.poll(); e.commit()
torch.cuda.synchronize()
nxt = e.cur ^ 1
op = None if e.operand is e.master else e.operand[nxt]
bias = None if e.bias is None else e.bias[nxt]
for _ in range(5):
    ops.normalize_loop_tail(e.sums, e.counts, e.master[e.cur], e.master[nxt], op, e.empty, e.shift2, bias, e.mind,
                            e._part, e.obj, e.changed, e.merges_it, e._flags_d, e._tail_ctr)
torch.cuda.synchronize()
print("ok")
