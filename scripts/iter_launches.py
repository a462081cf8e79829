"""A few pipelined Lloyd iterations (LloydEngine.run, CUDA graphs) at one BASELINE
config, for an ncu launch list of everything one iteration launches (dev aid).
usage: python scripts/iter_launches.py {2|3|4} [iters]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_09229_b200 import LloydEngine  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
B, N, K, d, dt = {"2": (1, 1 << 20, 1024, 128, torch.bfloat16), "3": (1, 1 << 23, 4096, 128, torch.bfloat16),
                  "4": (64, 16384, 256, 64, torch.float16)}[cfg]
g = torch.Generator(device="cuda").manual_seed(0)
centers = torch.rand((B, K, d), device="cuda", generator=g) * 20 - 10
lab = torch.randint(0, K, (B, N), device="cuda", generator=g)
x = (torch.gather(centers, 1, lab[..., None].expand(B, N, d))
     + torch.randn((B, N, d), device="cuda", generator=g)).to(dt).contiguous()
c0 = torch.stack([x[b, torch.randperm(N, device="cuda", generator=g)[:K]] for b in range(B)]).float()
eng = LloydEngine(x, K)
eng.set_centroids(c0)
h = torch.empty((64, B), dtype=torch.float64, device="cuda")
for _ in range(2):
    eng.run(4, -1.0, h, stop_on_repeat=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
eng.run(iters, -1.0, h, stop_on_repeat=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
