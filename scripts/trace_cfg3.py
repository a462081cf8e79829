"""In-kernel timeline of one config-3 FlashAssign (FK_ASSIGN_TRACE), plain and with the
engine's histogram fold + precomputed row norms (dev aid).  usage: python scripts/trace_cfg3.py [B N K d]"""
import os
import subprocess
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_09229_b200 import ops  # noqa: E402

B, N, K, d = (int(v) for v in sys.argv[1:5]) if len(sys.argv) > 4 else (1, 1 << 23, 4096, 128)
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn((B, N, d), device="cuda", generator=g).to(torch.bfloat16)
c = x[:, torch.randperm(N, device="cuda", generator=g)[:K]].contiguous()
fold = ops.hist_fold(x, K)
xn = ops.assign_row_norms(x, K)
for tag, kw in (("plain", {}), ("fold_xnorm", {"hist": fold, "xnorm": xn})):
    ops.assign(x, c, **kw)
    if "hist" in kw:
        fold.clear()
    path = f"gpurun_out/r02/trace_cfg3_{tag}.txt"
    os.environ["FK_ASSIGN_TRACE"] = path
    print("==", tag, flush=True)
    print(subprocess.run([sys.executable, "-c", f"""
import os, sys, torch
sys.path.insert(0, '.')
os.environ['FK_ASSIGN_TRACE'] = {path!r}
from paper_2603_09229_b200 import ops
B, N, K, d = {B}, {N}, {K}, {d}
g = torch.Generator(device='cuda').manual_seed(0)
x = torch.randn((B, N, d), device='cuda', generator=g).to(torch.bfloat16)
c = x[:, torch.randperm(N, device='cuda', generator=g)[:K]].contiguous()
kw = {{}}
if {tag!r} == 'fold_xnorm':
    kw = dict(hist=ops.hist_fold(x, K), xnorm=ops.assign_row_norms(x, K))
ops.assign(x, c, **kw)
torch.cuda.synchronize()
"""], capture_output=True, text=True).stderr[-500:])
    print(subprocess.run([sys.executable, "scripts/trace_assign.py", path], capture_output=True,
                         text=True).stdout[-600:], flush=True)
