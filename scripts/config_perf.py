"""Per-phase timing of one Lloyd iteration for BASELINE configs 2 and 4 (dev aid)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2603_09229_b200 import ops, LloydEngine

def run(name, B, N, K, d, dtype, reps=20):
    g = torch.Generator(device="cuda").manual_seed(0)
    centers = torch.rand((B, K, d), device="cuda", generator=g) * 20 - 10
    lab = torch.randint(0, K, (B, N), device="cuda", generator=g)
    x = (torch.gather(centers, 1, lab[..., None].expand(B, N, d)) + torch.randn((B, N, d), device="cuda", generator=g)).to(dtype).contiguous()
    c0 = torch.stack([x[b, torch.randperm(N, device="cuda", generator=g)[:K]] for b in range(B)]).float()
    eng = LloydEngine(x, K)
    eng.set_centroids(c0)
    for _ in range(3):
        eng.iterate(); eng.poll(); eng.commit()
    torch.cuda.synchronize()
    ev = lambda: torch.cuda.Event(enable_timing=True)
    s, e = ev(), ev()
    s.record()
    for _ in range(reps):
        eng.iterate(); eng.poll(); eng.commit()
    e.record(); torch.cuda.synchronize()
    t_it = s.elapsed_time(e) / reps
    def t(fn):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        a, b = ev(), ev(); a.record()
        for _ in range(reps): fn()
        b.record(); torch.cuda.synchronize()
        return a.elapsed_time(b) / reps
    slot = eng.it & 1
    ta = t(lambda: ops.assign(x, eng.operand[eng.cur], idx_out=eng.ids[slot], mind_out=eng.mind))
    tu = t(lambda: ops.update(x, eng.ids[slot], K, N, sums=eng.sums, counts=eng.counts))
    tn = t(lambda: ops.normalize(eng.sums, eng.counts, eng.master[eng.cur], out=eng.master[eng.cur ^ 1],
                                  operand_out=None if eng.operand is eng.master else eng.operand[eng.cur ^ 1],
                                  empty=eng.empty, shift2=eng.shift2))
    # pipelined loop (LloydEngine.run: next assign queued before the poll)
    def pipe(graphs):
        eng.use_graphs = graphs
        for _ in range(2):
            eng.run(4, -1.0, stop_on_repeat=False)  # warm: captures every (slot, centroid-slot) graph once
            eng.run(3, -1.0, stop_on_repeat=False)
        torch.cuda.synchronize()
        s2, e2 = ev(), ev()
        s2.record()
        its, _, _ = eng.run(reps, -1.0, stop_on_repeat=False)
        e2.record(); torch.cuda.synchronize()
        return s2.elapsed_time(e2) / its
    t_pipe = pipe(True)
    t_pipe_eager = pipe(False)
    fl = 2 * B * N * K * d
    by = B * N * d * x.element_size() + 4 * B * N + 4 * B * K * d + 4 * B * K
    print(f"{name}: iteration {t_it*1e3:.1f} us (pipelined {t_pipe*1e3:.1f} us graphs, {t_pipe_eager*1e3:.1f} us eager) | assign {ta*1e3:.1f} us ({fl/ta/1e9:.0f} TF/s) | "
          f"update {tu*1e3:.1f} us ({by/tu/1e6:.0f} GB/s) | normalize {tn*1e3:.1f} us | "
          f"{B*N/(t_it*1e-3)/1e9:.2f} Gpoints/s")

run("cfg2 N=1M d=128 K=1024 bf16", 1, 1 << 20, 1024, 128, torch.bfloat16)
run("cfg4 B=64 N=16k d=64 K=256 fp16", 64, 16384, 256, 64, torch.float16)
run("cfg4-bf16", 64, 16384, 256, 64, torch.bfloat16)
run("cfg3 N=8M d=128 K=4096 bf16", 1, 1 << 23, 4096, 128, torch.bfloat16, reps=5)
