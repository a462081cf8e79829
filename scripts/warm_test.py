"""Warm-start assign: parity vs cold and timing over Lloyd iterations (dev aid)."""
import sys, os, torch, time
sys.path.insert(0, ".")
import numpy as np
from paper_2603_09229_b200 import ops, LloydEngine
N, K, d = 1 << 23, 4096, 128
g = torch.Generator(device="cuda").manual_seed(0)
centers = torch.rand((K, d), device="cuda", generator=g) * 20 - 10
lab = torch.randint(0, K, (N,), device="cuda", generator=g)
x = (centers[lab] + torch.randn((N, d), device="cuda", generator=g)).to(torch.bfloat16)[None].contiguous()
c0 = x[:, torch.randperm(N, device="cuda", generator=g)[:K]].float()
eng = LloydEngine(x, K)
eng.set_centroids(c0)
ev = lambda: torch.cuda.Event(enable_timing=True)
for it in range(12):
    slot = eng.it & 1
    prev = eng.ids[slot ^ 1].clone() if it > 0 else None
    s, e = ev(), ev()
    s.record()
    eng.iterate()
    e.record(); torch.cuda.synchronize()
    # cold reference assign for the same centroids
    c_op = eng.operand[eng.cur]
    ids_cold, mind_cold = ops.assign(x, c_op)
    ids_w = eng.ids[slot]
    diff = (ids_w != ids_cold).sum().item()
    # time warm vs cold assign alone
    t = []
    for mode in ("warm", "cold"):
        ss, ee = ev(), ev()
        ss.record()
        for _ in range(3):
            if mode == "warm" and prev is not None:
                fl = torch.zeros((), dtype=torch.int32, device="cuda")
                ops.assign(x, c_op, idx_prev=prev, changed=fl)
            else:
                ops.assign(x, c_op)
        ee.record(); torch.cuda.synchronize()
        t.append(ss.elapsed_time(ee) / 3)
    md = (eng.mind - mind_cold).abs().max().item()
    print(f"it {it}: iter {s.elapsed_time(e):.3f} ms  assign warm {t[0]:.3f} cold {t[1]:.3f} ms  id diffs vs cold {diff}  max|dmind| {md:.3g}")
    eng.commit()
