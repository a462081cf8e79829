"""f32/f64 assign: certified tensor-core path vs the exact CUDA-core mirror vs
the cuBLAS materializing foil; f64 update: serial (bitwise) vs slice-parallel.
Device-timed (CUDA events, median of reps)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_09229_b200 import ops  # noqa: E402


def tm(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def blobs(N, K, d, dt, g):
    centers = torch.rand((K, d), device="cuda", generator=g) * 20 - 10
    lab = torch.randint(0, K, (N,), device="cuda", generator=g)
    x = centers[lab] + torch.randn((N, d), device="cuda", generator=g)
    return x[None].to(dt)



def main():
  g = torch.Generator(device="cuda").manual_seed(0)
  for (N, K, d, dt, data) in [(65536, 1024, 128, torch.float32, "gauss"), (65536, 1024, 128, torch.float32, "blobs"),
                              (1 << 20, 1024, 128, torch.float32, "blobs"), (1 << 20, 1024, 128, torch.float64, "blobs"),
                              (1 << 23, 4096, 128, torch.float32, "blobs"), (1 << 20, 1024, 128, torch.float32, "gauss")]:
      x = blobs(N, K, d, dt, g) if data == "blobs" else torch.randn((1, N, d), device="cuda", generator=g, dtype=dt)
      c = x[:, torch.randperm(N, device="cuda", generator=g)[:K]].clone()
      xs = ops.assign_xsplit(x)
      t_xs = tm(lambda: ops.assign_xsplit(x, out=xs))
      ids = torch.empty((1, N), dtype=torch.int32, device="cuda")
      mind = torch.empty((1, N), dtype=dt, device="cuda")
      t_split = tm(lambda: ops.assign(x, c, xsplit=xs, idx_out=ids, mind_out=mind))
      ids_s = ids.clone()
      fb = ops.split_fallback_rows(x, K)[0]
      flops = 2.0 * N * K * d
      line = (f"{data} N={N} K={K} d={d} {str(dt)[6:]}: split {t_split*1e3:8.1f} us "
              f"({flops / t_split / 1e9:6.1f} TF/s-equiv, fallback {fb} rows = {100.0 * fb / N:.2f}%) | xsplit {t_xs*1e3:7.1f} us")
      if N * K <= (1 << 30):
          t_mir = tm(lambda: ops.assign(x, c, path="mirror", idx_out=ids, mind_out=mind), reps=3)
          assert torch.equal(ids, ids_s), "split != mirror"
          xf, cf = x[0], c[0]
          def foil():
              dd = (xf * xf).sum(1, keepdim=True) + (cf * cf).sum(1)[None] - 2.0 * (xf @ cf.T)
              return dd.argmin(1)
          t_foil = tm(foil, reps=3)
          line += f" | mirror {t_mir*1e3:9.1f} us | cuBLAS foil {t_foil*1e3:8.1f} us"
      print(line, flush=True)
      if dt == torch.float64:
          for env in ("serial", "parallel"):
              pass
      del x, xs, c, ids, mind
      torch.cuda.empty_cache()


if __name__ == '__main__':
    main()
