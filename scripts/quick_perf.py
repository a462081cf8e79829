"""Quick CUDA-event timing of the hot-path kernels at BASELINE config 3 (dev aid)."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2603_09229_b200 import ops

def timeit(fn, reps=10, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 23
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
d = 128
torch.manual_seed(0)
x = (torch.randn(1, N, d, device="cuda") + torch.randint(-10, 10, (1, 1, d), device="cuda")).to(torch.bfloat16)
c = x[:, torch.randperm(N, device="cuda")[:K]].contiguous()
ids, mind = ops.assign(x, c)
t_a = timeit(lambda: ops.assign(x, c, idx_out=ids, mind_out=mind))
fl = 2.0 * N * K * d
print(f"assign  N={N} K={K}: {t_a:.3f} ms  {fl/t_a/1e9:.1f} TFLOP/s  ({fl/t_a/1e9/1654.1*100:.1f}% of 1654 burst)")
sums, counts = ops.update(x, ids, K, N)
t_u = timeit(lambda: ops.update(x, ids, K, N, sums=sums, counts=counts))
by = N * d * 2 + 4 * N + 4 * K * d + 4 * K
print(f"update: {t_u:.3f} ms  {by/t_u/1e6:.1f} GB/s ({by/t_u/1e6/6532.9*100:.1f}% of 6533)")
prev = c.float()
t_n = timeit(lambda: ops.normalize(sums, counts, prev, operand_dtype=torch.bfloat16))
print(f"normalize: {t_n:.3f} ms")
t_o = timeit(lambda: ops.objective(mind))
print(f"objective: {t_o:.3f} ms")
t_s = timeit(lambda: ops.scatter(x, ids, K), reps=3, warm=1)
print(f"scatter foil: {t_s:.3f} ms")
