import sys, torch
sys.path.insert(0, ".")
from paper_2603_09229_b200 import ops
B, N, K, d = 64, 16384, 256, 64
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn((B, N, d), device="cuda", generator=g).to(torch.float16)
c = x[:, :K].contiguous()
for _ in range(3):
    ops.assign(x, c)
torch.cuda.synchronize()
