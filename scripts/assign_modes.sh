for m in ${MODES:-0 1 2}; do FK_ASSIGN_DEBUG_MODE=$m python - <<'PY'
import os, sys, torch
sys.path.insert(0, ".")
from paper_2603_09229_b200 import ops
N, K, d = 1 << 23, 4096, 128
torch.manual_seed(0)
x = (torch.randn(1, N, d, device="cuda")).to(torch.bfloat16)
c = x[:, :K].contiguous()
ids, mind = ops.assign(x, c)
for _ in range(3): ops.assign(x, c, idx_out=ids, mind_out=mind)
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(10): ops.assign(x, c, idx_out=ids, mind_out=mind)
e.record(); torch.cuda.synchronize()
t = s.elapsed_time(e) / 10
print("mode", os.environ["FK_ASSIGN_DEBUG_MODE"], f"{t:.3f} ms", f"{2*N*K*d/t/1e9:.0f} TF/s-equiv")
PY
done
