"""compute-sanitizer driver for the update + normalize kernels (block and staged scatter paths; dev aid)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2603_09229_b200 import ops
torch.manual_seed(0)
for (B, N, K, d, dt) in [(1, 40000, 1000, 64, torch.bfloat16), (2, 20000, 300, 32, torch.float16),
                         (1, 17000, 4096, 16, torch.float32), (1, 131072, 4096, 16, torch.bfloat16),
                         (3, 50001, 777, 8, torch.float32)]:
    x = torch.randn(B, N, d, device="cuda").to(dt)
    ids = torch.randint(0, K, (B, N), device="cuda", dtype=torch.int32)
    sums, counts = ops.update(x, ids, K, 4096)
    c = x[:, :K].float().contiguous()
    out, op, empty = ops.normalize(sums, counts, c, operand_dtype=dt if dt != torch.float32 else None)
    torch.cuda.synchronize()
    assert int(counts.sum()) == B * N
print("ok")
