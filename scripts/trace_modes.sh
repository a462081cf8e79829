mkdir -p gpurun_out
for m in 0 1; do
FK_ASSIGN_DEBUG_MODE=$m bash scripts/clock_probe.sh mode$m
FK_ASSIGN_DEBUG_MODE=$m python - <<'PY'
import os, sys, torch
sys.path.insert(0, ".")
from paper_2603_09229_b200 import ops
N, K, d = 1 << 23, 4096, 128
torch.manual_seed(0)
x = torch.randn(1, N, d, device="cuda").to(torch.bfloat16)
c = x[:, :K].contiguous()
ids, mind = ops.assign(x, c)
for _ in range(20): ops.assign(x, c, idx_out=ids, mind_out=mind)
os.environ["FK_ASSIGN_TRACE"] = "gpurun_out/trace.txt"
ops.assign(x, c, idx_out=ids, mind_out=mind)
PY
echo "== trace mode $m"; python scripts/trace_assign.py gpurun_out/trace.txt | tail -4
done
