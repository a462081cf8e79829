"""BASELINE config 5 at its per-GPU size: one out-of-core Lloyd pass over this
GPU's shard of the 2e9-point fp16 dataset (2e9 / 8 = 250M points, d=128,
K=65536) streamed from pinned host memory through the public API
(paper_2603_09229_b200.out_of_core_iteration over a HostStream: copy stream +
two device buffers).  Reports the pass time, the achieved H2D rate, the
assign rate, and how much of the pass the copy costs beyond compute (copy-only
and compute-only references measured on the same data).
usage: python scripts/cfg5_shard.py [points] [chunk_points]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2603_09229_b200 as fk  # noqa: E402
from paper_2603_09229_b200 import ops  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 250_000_000
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 23
K, d = 65536, 128
t0 = time.perf_counter()
host = torch.empty((1, N, d), dtype=torch.float16).pin_memory()
t_pin = time.perf_counter() - t0
g = torch.Generator(device="cuda").manual_seed(0)
centers = torch.rand((K // 16, d), device="cuda", generator=g) * 20 - 10
for lo in range(0, N, chunk):  # generated on the GPU, landed in pinned host memory
    hi = min(N, lo + chunk)
    lab = torch.randint(0, K // 16, (hi - lo,), device="cuda", generator=g)
    host[0, lo:hi].copy_((centers[lab] + torch.randn((hi - lo, d), device="cuda", generator=g)).half())
torch.cuda.synchronize()
print(f"shard: {N} points x {d} fp16 = {N * d * 2 / 1e9:.1f} GB pinned ({t_pin:.1f} s to pin)", flush=True)
idx = torch.randperm(N, generator=torch.Generator().manual_seed(1))[:K]
c0 = fk.Centroids(host[:, idx].float().cuda(), check_finite=False)
stream = fk.HostStream(host, chunk, pin=False)
cfg = fk.KMeansConfig(K, max_iters=1, precision="fp16")
counters = fk.Counters()
c1, store, _ = fk.out_of_core_iteration(stream, c0, cfg, counters)  # warm-up pass
torch.cuda.synchronize()
flops = 2.0 * N * K * d
for it in range(2):
    t0 = time.perf_counter()
    c1, store, _ = fk.out_of_core_iteration(stream, c0, cfg, counters, store=store)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"pass {it}: {dt:.3f} s | H2D {N * d * 2 / dt / 1e9:.1f} GB/s | {N / dt / 1e6:.1f} M points/s | "
          f"assign-equivalent {flops / dt / 1e12:.0f} TFLOP/s", flush=True)
# copy-only and compute-only references on the same data
buf = torch.empty((chunk, d), dtype=torch.float16, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for lo in range(0, N, chunk):
    n = min(chunk, N - lo)
    buf[:n].copy_(host[0, lo:lo + n], non_blocking=True)
torch.cuda.synchronize()
t_copy = time.perf_counter() - t0
xs = host[:, :chunk].cuda()
cop = c0.data.half()
ops.assign(xs, cop)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(2):
    ids, _ = ops.assign(xs, cop)
    ops.update(xs, ids, K, chunk)
ev[1].record()
torch.cuda.synchronize()
t_chunk = ev[0].elapsed_time(ev[1]) / 2e3
t_comp = t_chunk * N / chunk
print(f"copy-only {t_copy:.3f} s ({N * d * 2 / t_copy / 1e9:.1f} GB/s); assign+update per {chunk}-point chunk "
      f"{t_chunk * 1e3:.1f} ms -> compute-only {t_comp:.3f} s; pass / compute-only = {dt / t_comp:.3f} "
      f"(copy hidden: {max(0.0, 1 - (dt - t_comp) / t_copy) * 100:.0f}%)", flush=True)
print("ok")
