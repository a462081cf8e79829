"""f64 update: time of ops.update (serial bitwise segsum by default; run with
FK_SEGSUM_F64=parallel for the slice-parallel variant)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_09229_b200 import ops  # noqa: E402
from scripts.split_perf import tm  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
for N, K, d, chunk in [(1 << 20, 1024, 128, 1 << 15), (1 << 23, 4096, 128, 1 << 18), (1 << 20, 16, 64, 1 << 15),
                       (10000, 8, 16, 256)]:
    x = torch.randn((1, N, d), device="cuda", generator=g, dtype=torch.float64)
    ids = torch.randint(0, K, (1, N), device="cuda", generator=g, dtype=torch.int32)
    t = tm(lambda: ops.update(x, ids, K, chunk))
    byt = N * d * 8 + N * 4
    print(f"{os.environ.get('FK_SEGSUM_F64', 'serial')} N={N} K={K} d={d} chunk={chunk}: update {t*1e3:8.1f} us "
          f"({byt / t / 1e6:7.1f} GB/s algorithmic)", flush=True)
