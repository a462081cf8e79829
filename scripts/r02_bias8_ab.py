"""fp8 bias step A/B (FK_ASSIGN_BIAS8=1) -- dev aid.

usage: FK_ASSIGN_BIAS8=0|1 python scripts/r02_bias8_ab.py out.npz   (times + saves ids/min_dists)
       python scripts/r02_bias8_ab.py --compare a.npz b.npz        (ids / min_dists differences)
       python scripts/r02_bias8_ab.py --grid                         (integer grid vs the oracle, bitwise)
"""
import sys, numpy as np, torch
sys.path.insert(0, ".")

if sys.argv[1] == "--compare":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    for k in sorted(a.files):
        if k.startswith("ids"):
            print(k, "id mismatches:", int((a[k] != b[k]).sum()), "of", a[k].size)
        else:
            m0, m1 = a[k].astype(np.float64), b[k].astype(np.float64)
            rel = np.abs(m0 - m1) / np.maximum(np.abs(m0), 1e-30)
            print(k, "min_dists bitwise equal:", bool(np.array_equal(a[k], b[k])), "max rel diff %.3g" % rel.max())
    sys.exit(0)

from paper_2603_09229_b200 import ops
if sys.argv[1] == "--grid":
    from oracle import oracle as O
    for i, (B, N, K, d, dt) in enumerate([(1, 5000, 1000, 128, torch.bfloat16), (2, 3000, 300, 64, torch.float16),
                                          (64, 2048, 256, 64, torch.float16)]):
        g = torch.Generator().manual_seed(7 + i)
        x = torch.randint(-8, 9, (B, N, d), generator=g).to(dt)
        c = torch.randint(-8, 9, (B, K, d), generator=g).to(dt)
        a, m = ops.assign(x.cuda(), c.cuda())
        ar, mr = O.assign(x.float().numpy(), c.float().numpy())
        print("grid", (B, N, K, d), "ids equal:", bool(np.array_equal(a.cpu().numpy(), ar)),
              "min_dists equal:", bool(np.array_equal(m.cpu().numpy(), mr)))
    sys.exit(0)

shapes = [(1, 8388608, 4096, 128, torch.bfloat16), (1, 1048576, 1024, 128, torch.bfloat16),
          (64, 16384, 256, 64, torch.float16)]
out = {}
for i, (B, N, K, d, dt) in enumerate(shapes):
    g = torch.Generator(device="cuda").manual_seed(1)
    centers = torch.rand((B, K, d), device="cuda", generator=g) * 20 - 10
    lab = torch.randint(0, K, (B, N), device="cuda", generator=g)
    x = (torch.gather(centers, 1, lab[..., None].expand(B, N, d))
         + torch.randn((B, N, d), device="cuda", generator=g)).to(dt).contiguous()
    c = torch.stack([x[b, torch.randperm(N, device="cuda", generator=g)[:K]] for b in range(B)]).contiguous()
    ids, mind = ops.assign(x, c)
    torch.cuda.synchronize()
    sub = slice(0, 1 << 20)
    out[f"ids{i}"] = ids.reshape(-1)[sub].cpu().numpy()
    out[f"mind{i}"] = mind.reshape(-1)[sub].cpu().numpy()
    it = 20 if N * K > 1e9 else 200
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
    print(f"B={B} N={N} K={K} d={d}: {t*1e3:8.1f} us (incl. the operand build) {2*B*N*K*d/t/1e9:6.0f} TF/s", flush=True)
np.savez(sys.argv[1], **out)
