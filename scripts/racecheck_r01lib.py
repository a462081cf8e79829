"""Round-1 library (ablib/libflashkmeans_r01.so) FlashAssign under racecheck, direct ctypes
(dev aid: is the tcgen05.alloc hazard report pre-existing?)."""
import ctypes
import torch
L = ctypes.CDLL("ablib/libflashkmeans_r01.so")
P, I64, SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t
L.fk_assign_workspace.restype = SZ
L.fk_assign_workspace.argtypes = [ctypes.c_int, I64, I64, I64, I64]
L.fk_assign.restype = ctypes.c_int
L.fk_assign.argtypes = [ctypes.c_int, P, P, I64, I64, I64, I64, P, P, P, P, P, SZ, P]
B, N, K, d = 1, 3000, 1000, 128
x = torch.randn(B, N, d, device="cuda").to(torch.bfloat16)
c = x[:, :K].contiguous()
ids = torch.empty((B, N), dtype=torch.int32, device="cuda")
mind = torch.empty((B, N), dtype=torch.float32, device="cuda")
ws = torch.empty(L.fk_assign_workspace(1, B, N, K, d), dtype=torch.uint8, device="cuda")
st = L.fk_assign(1, x.data_ptr(), c.data_ptr(), B, N, K, d, ids.data_ptr(), mind.data_ptr(), None, None,
                 ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("status", st)
