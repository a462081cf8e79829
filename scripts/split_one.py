"""One certified f32 assign at N=1M, K=1024, d=128 (blobs) for an ncu launch list."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_09229_b200 import ops  # noqa: E402
from scripts.split_perf import blobs  # noqa: E402
g = torch.Generator(device="cuda").manual_seed(0)
N, K, d = 1 << 20, 1024, 128
x = blobs(N, K, d, torch.float32, g) if sys.argv[1:2] != ["gauss"] else torch.randn((1, N, d), device="cuda", generator=g)
c = x[:, torch.randperm(N, device="cuda", generator=g)[:K]].clone()
xs = ops.assign_xsplit(x)
ops.assign(x, c, xsplit=xs)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
ops.assign(x, c, xsplit=xs)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
