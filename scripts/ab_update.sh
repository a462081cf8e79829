# A/B the update path of two library builds on the same box
for r in 1 2; do for lib in "$1" "$2"; do
FK_LIB_PATH=$lib python - <<'PY'
import os, sys, torch
sys.path.insert(0, ".")
from paper_2603_09229_b200 import ops
N, K, d = 1 << 23, 4096, 128
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn((1, N, d), device="cuda", generator=g).to(torch.bfloat16)
ids = torch.randint(0, K, (1, N), device="cuda", generator=g, dtype=torch.int32)
s, c = ops.update(x, ids, K, N)
for _ in range(3): ops.update(x, ids, K, N, sums=s, counts=c)
torch.cuda.synchronize()
a, b = torch.cuda.Event(True), torch.cuda.Event(True)
a.record()
for _ in range(20): ops.update(x, ids, K, N, sums=s, counts=c)
b.record(); torch.cuda.synchronize()
print(os.path.basename(os.environ["FK_LIB_PATH"]), f"update {a.elapsed_time(b)/20*1e3:.1f} us")
PY
done; done
