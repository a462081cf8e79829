"""One FlashAssign launch on config-3 blob data (for ncu capture; dev aid)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2603_09229_b200 import ops
N, K, d = 1 << 23, 4096, 128
g = torch.Generator(device="cuda").manual_seed(0)
centers = torch.rand((K, d), device="cuda", generator=g) * 20 - 10
lab = torch.randint(0, K, (N,), device="cuda", generator=g)
x = (centers[lab] + torch.randn((N, d), device="cuda", generator=g)).to(torch.bfloat16)[None].contiguous()
c = x[:, torch.randperm(N, device="cuda", generator=g)[:K]].contiguous()
for _ in range(3):
    ids, mind = ops.assign(x, c)
torch.cuda.synchronize()
