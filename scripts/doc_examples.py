"""Run the code examples of README.md and INTEGRATION.md on a GPU (doc check)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, ".")

# README quick start
import paper_2603_09229_b200 as fm
x = fm.generate_dataset(1, 1 << 20, 1024, 128, 1.0, 0, precision="bf16")
res = fm.lloyd_run(fm.DataMatrix(x.data.cuda()), fm.KMeansConfig(1024, max_iters=20, init="kmeanspp"))
print("README lloyd_run kmeanspp:", res.iterations_run, "iterations")

# INTEGRATION option A
r = fm.lloyd_run(fm.DataMatrix(x.data.cuda()), fm.KMeansConfig(1024, max_iters=20))
c = fm.init_centroids(x, 1024, 0)
a, mind, counters = fm.flash_assign(x, c, fm.TilingConfig(128, 256, 1 << 20), fm.Counters())
stats, counters = fm.sort_inverse_update(x, a, 1024, 1 << 20, counters)
new_c, empty = fm.normalize(stats, c)
print("option A:", r.iterations_run, a.numpy().shape, counters.synchronized_merges, len(empty[0]))

# INTEGRATION option B (ctypes stub), against the in-tree library
_L = ctypes.CDLL(os.path.join("paper_2603_09229_b200", "_lib", "libflashkmeans.so"))
_P, _I64, _SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t
_L.fk_assign_workspace.restype = _SZ
_L.fk_assign_workspace.argtypes = [ctypes.c_int, _I64, _I64, _I64, _I64]
_L.fk_assign.restype = ctypes.c_int
_L.fk_assign.argtypes = [ctypes.c_int, _P, _P, _I64, _I64, _I64, _I64, _P, _P, _P, _P, _P, _SZ, _P]
FK = {torch.float32: 0, torch.bfloat16: 1, torch.float16: 2, torch.float64: 3}

def flash_assign_b200(x, c):
    B, N, d = x.shape; K = c.shape[1]; dt = FK[x.dtype]
    ids = torch.empty((B, N), dtype=torch.int32, device=x.device)
    mind = torch.empty((B, N), dtype=torch.float32 if dt in (1, 2) else x.dtype, device=x.device)
    ws = torch.empty(_L.fk_assign_workspace(dt, B, N, K, d), dtype=torch.uint8, device=x.device)
    st = _L.fk_assign(dt, x.data_ptr(), c.data_ptr(), B, N, K, d, ids.data_ptr(), mind.data_ptr(),
                      None, None, ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream)
    if st == 1: raise ValueError("fk_assign: invalid argument")
    if st: raise RuntimeError(f"fk_assign failed ({st})")
    return ids, mind

ids, md = flash_assign_b200(x.data.cuda(), c.data.cuda())
assert torch.equal(ids.cpu(), a.values.cpu())
print("option B stub == drop-in flash_assign")

# INTEGRATION k-means++ stub
_L.fk_kmeanspp_workspace.restype = _SZ
_L.fk_kmeanspp_workspace.argtypes = [_I64, _I64, _I64, _I64]
_L.fk_kmeanspp.restype = ctypes.c_int
_L.fk_kmeanspp.argtypes = [ctypes.c_int, _P, _I64, _I64, _I64, _I64, _P, _P, _P, _P, _P, _SZ, _P]

def kmeanspp_indices_b200(x, k, seed):
    B, N, d = x.shape
    rngs = [np.random.default_rng((seed, b)) for b in range(B)]
    first = [r.integers(N) for r in rngs]
    u = np.stack([r.random(k - 1) for r in rngs])
    idx = torch.zeros((B, k), dtype=torch.int64, device=x.device); idx[:, 0] = torch.tensor(first)
    halted = torch.empty(B, dtype=torch.int32, device=x.device)
    m = torch.empty((B, N), dtype=torch.float64, device=x.device)
    ws = torch.empty(_L.fk_kmeanspp_workspace(B, N, k, d), dtype=torch.uint8, device=x.device)
    ud = torch.from_numpy(u).to(x.device)
    st = _L.fk_kmeanspp(FK[x.dtype], x.data_ptr(), B, N, d, k, ud.data_ptr(), idx.data_ptr(),
                        halted.data_ptr(), m.data_ptr(), ws.data_ptr(), ws.numel(),
                        torch.cuda.current_stream().cuda_stream)
    if st == 1: raise ValueError("fk_kmeanspp: invalid argument")
    idx, halted = idx.cpu().numpy(), halted.cpu().numpy()
    for b in range(B):
        if halted[b] < k:
            r = np.random.default_rng((seed, b)); r.integers(N); r.random(halted[b] - 1)
            idx[b, halted[b]:] = [r.integers(N) for _ in range(halted[b], k)]
    return idx

from paper_2603_09229_b200.core import kmeanspp_indices_device
xs = x.data[:, :100000].contiguous().cuda()
assert np.array_equal(kmeanspp_indices_b200(xs, 64, 3), kmeanspp_indices_device(xs, 64, 3))
print("k-means++ stub == device seeding")
