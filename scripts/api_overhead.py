"""Where the API-level update time goes at config 2 (dev aid)."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2603_09229_b200 as fk
from paper_2603_09229_b200 import ops

N, K, d = 1 << 20, 1024, 128
x = fk.generate_dataset(1, N, K, d, 1.0, 0, "bf16")
x = fk.DataMatrix(x.data.cuda(), check_finite=False)
c = fk.init_centroids(x, K, 0)
a, _, _ = fk.flash_assign(x, c, fk.TilingConfig(64, 128, 16384), fk.Counters())

def dev_ms(fn, reps=20):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); fn(); e.record(); e.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort(); return ts[len(ts) // 2] * 1e3

def host_us(fn, reps=20):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    ts.sort(); return ts[len(ts) // 2] * 1e6

sums = torch.empty((1, K, d), dtype=torch.float64, device="cuda")
counts = torch.empty((1, K), dtype=torch.int64, device="cuda")
m = torch.zeros((), dtype=torch.int64, device="cuda")
print(f"ops.update (preallocated)   dev {dev_ms(lambda: ops.update(x.data, a.values, K, 16384, sums=sums, counts=counts, merges=m)):8.1f} us")
print(f"ops.update (alloc)          dev {dev_ms(lambda: ops.update(x.data, a.values, K, 16384, merges=m)):8.1f} us")
print(f"aminmax+tolist              dev {dev_ms(lambda: torch.stack(torch.aminmax(a.values)).tolist()):8.1f} us")
print(f"sort_inverse_update         dev {dev_ms(lambda: fk.sort_inverse_update(x, a, K, 16384, fk.Counters())):8.1f} us  host {host_us(lambda: fk.sort_inverse_update(x, a, K, 16384, fk.Counters())):8.1f} us")
print(f"flash_assign                dev {dev_ms(lambda: fk.flash_assign(x, c, fk.TilingConfig(64, 128, 16384), fk.Counters())):8.1f} us  host {host_us(lambda: fk.flash_assign(x, c, fk.TilingConfig(64, 128, 16384), fk.Counters())):8.1f} us")
ids = torch.empty((1, N), dtype=torch.int32, device="cuda"); md = torch.empty((1, N), device="cuda")
print(f"ops.assign (preallocated)   dev {dev_ms(lambda: ops.assign(x.data, c.data, idx_out=ids, mind_out=md)):8.1f} us")
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    ops.assign(x.data, c.data, idx_out=ids, mind_out=md)
print(f"ops.assign (graph replay)   dev {dev_ms(lambda: g.replay()):8.1f} us")
g2 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g2):
    ops.update(x.data, a.values, K, 16384, sums=sums, counts=counts, merges=m)
print(f"ops.update (graph replay)   dev {dev_ms(lambda: g2.replay()):8.1f} us")
