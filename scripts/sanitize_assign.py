"""compute-sanitizer driver for FlashAssign (pair kernel: alternate-tile and column-split epilogues; dev aid)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2603_09229_b200 import ops
torch.manual_seed(0)
for (B, N, K, d, dt) in [(1, 3000, 1000, 128, torch.bfloat16), (2, 1500, 200, 64, torch.float16),
                         (1, 777, 4096, 256, torch.bfloat16), (3, 513, 33, 24, torch.bfloat16)]:
    x = torch.randn(B, N, d, device="cuda").to(dt)
    c = x[:, :K].contiguous() if K <= N else torch.randn(B, K, d, device="cuda").to(dt)
    ids, mind = ops.assign(x, c)
    prev = ids.clone()
    changed = torch.zeros((), dtype=torch.int32, device="cuda")
    ids2, mind2 = ops.assign(x, c, idx_prev=prev, changed=changed)
    torch.cuda.synchronize()
    assert torch.equal(ids, ids2) and int(changed) == 0
print("ok")
