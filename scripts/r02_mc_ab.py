"""A/B of the multicast-quad FlashAssign (FK_ASSIGN_MC=1) against the pair kernel (dev aid).

usage: FK_ASSIGN_MC=0|1 python scripts/r02_mc_ab.py -> one line per shape: time, hash of (ids, min_dists)
"""
import hashlib, sys, torch
sys.path.insert(0, ".")
from paper_2603_09229_b200 import ops

shapes = [(1, 8388608, 4096, 128, torch.bfloat16), (1, 1048576, 1024, 128, torch.bfloat16),
          (1, 1048576 + 300, 529, 64, torch.float16), (1, 4096 * 5 + 256 + 7, 1024, 256, torch.bfloat16),
          (1, 1000, 700, 128, torch.bfloat16), (2, 65536, 1024, 128, torch.bfloat16)]
import os
sel = os.environ.get("SHAPES")
if sel:
    shapes = [shapes[int(i)] for i in sel.split(",")]
for B, N, K, d, dt in shapes:
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(B, N, d, device="cuda", generator=g).to(dt)
    c = torch.randn(B, K, d, device="cuda", generator=g).to(dt)
    ids, mind = ops.assign(x, c)
    torch.cuda.synchronize()
    h = hashlib.sha1(ids.cpu().numpy().tobytes() + mind.cpu().numpy().tobytes()).hexdigest()[:12]
    it = 40 if N * K > 1e9 else 400
    for _ in range(3):
        ops.assign(x, c, idx_out=ids, mind_out=mind)
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(it):
        ops.assign(x, c, idx_out=ids, mind_out=mind)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / it
    print(f"B={B} N={N} K={K} d={d} {str(dt)[6:]}: {t*1e3:8.1f} us {2*B*N*K*d/t/1e9:6.0f} TF/s hash {h}", flush=True)
