import sys, torch
sys.path.insert(0, ".")
from paper_2603_09229_b200 import LloydEngine
B, N, K, d = 64, 16384, 256, 64
g = torch.Generator(device="cuda").manual_seed(0)
centers = torch.rand((B, K, d), device="cuda", generator=g) * 20 - 10
lab = torch.randint(0, K, (B, N), device="cuda", generator=g)
x = (torch.gather(centers, 1, lab[..., None].expand(B, N, d)) + torch.randn((B, N, d), device="cuda", generator=g)).to(torch.float16).contiguous()
c0 = torch.stack([x[b, torch.randperm(N, device="cuda", generator=g)[:K]] for b in range(B)]).float()
eng = LloydEngine(x, K); eng.use_graphs = False
eng.set_centroids(c0)
for _ in range(4):
    eng.iterate(); eng.poll(); eng.commit()
torch.cuda.synchronize()
