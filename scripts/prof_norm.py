"""One normalize at config 4 (for an ncu capture; dev aid)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2603_09229_b200 import ops
B, K, d = 64, 256, 64
sums = torch.randn(B, K, d, dtype=torch.float64, device="cuda") * 1000
counts = torch.randint(1, 100, (B, K), dtype=torch.int64, device="cuda")
prev = torch.randn(B, K, d, device="cuda")
out = torch.empty_like(prev)
op = torch.empty(B, K, d, dtype=torch.float16, device="cuda")
empty = torch.empty(B, K, dtype=torch.uint8, device="cuda")
import os
sh = None if os.environ.get("NOSHIFT") else torch.zeros((), dtype=torch.float64, device="cuda")
for _ in range(5):
    ops.normalize(sums, counts, prev, out=out, operand_out=op, empty=empty, shift2=sh)
torch.cuda.synchronize()
