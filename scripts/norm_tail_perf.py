"""Warm per-launch time of the end-of-iteration kernels at BASELINE config 4
(and 2): plain normalize, normalize + objective + loop tail (one launch), and
the objective alone (dev aid).  usage: python scripts/norm_tail_perf.py"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_09229_b200 import LloydEngine, ops  # noqa: E402


def t(fn, reps=20, replays=20):
    """device time per call: reps calls captured in one CUDA graph (no host
    launch overhead in the number), replayed"""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(replays):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / (reps * replays) * 1e3


for name, (B, N, K, d, dt) in {"cfg4": (64, 16384, 256, 64, torch.float16),
                               "cfg2": (1, 1 << 20, 1024, 128, torch.bfloat16),
                               "cfg3": (1, 1 << 23, 4096, 128, torch.bfloat16),
                               "B8-N1M-K256": (8, 1 << 20, 256, 64, torch.bfloat16)}.items():
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn((B, N, d), device="cuda", generator=g).to(dt)
    eng = LloydEngine(x, K)
    eng.set_centroids(x[:, :K].float())
    eng.iterate(); eng.poll(); eng.commit()
    torch.cuda.synchronize()
    e = eng
    nxt = e.cur ^ 1
    op = None if e.operand is e.master else e.operand[nxt]
    bias = None if e.bias is None else e.bias[nxt]
    tn = t(lambda: ops.normalize(e.sums, e.counts, e.master[e.cur], out=e.master[nxt], operand_out=op,
                                 empty=e.empty, shift2=e.shift2))
    tt = t(lambda: ops.normalize_loop_tail(e.sums, e.counts, e.master[e.cur], e.master[nxt], op, e.empty,
                                           e.shift2, bias, e.mind, e._part, e.obj, e.changed, e.merges_it,
                                           e._flags_d, e._tail_ctr))
    to = t(lambda: ops.objective(e.mind, out=e.obj))

    def three():  # the unfused end of an iteration: normalize, partials, loop tail
        ops.normalize(e.sums, e.counts, e.master[e.cur], out=e.master[nxt], operand_out=op, empty=e.empty,
                      shift2=e.shift2)
        ops.objective_partials(e.mind, e._part)
        ops.loop_tail(e._part, B, N, e.obj, e.changed, e.shift2, e.merges_it, e._flags_d)
    t3 = t(three)
    print(f"{name}: normalize {tn:.1f} us | normalize+tail (one launch) {tt:.1f} us | objective {to:.1f} us | "
          f"normalize + partials + loop tail (3 launches) {t3:.1f} us", flush=True)
