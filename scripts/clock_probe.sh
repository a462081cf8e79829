# assign kernel alone for ~3 s with nvidia-smi sampling (dev aid)
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 50 > gpurun_out/clk_$1.csv &
P=$!
sleep 0.5
python - <<'PY'
import sys, torch, time
sys.path.insert(0, ".")
from paper_2603_09229_b200 import ops
N, K, d = 1 << 23, 4096, 128
g = torch.Generator(device="cuda").manual_seed(0)
centers = torch.rand((K, d), device="cuda", generator=g) * 20 - 10
lab = torch.randint(0, K, (N,), device="cuda", generator=g)
x = (centers[lab] + torch.randn((N, d), device="cuda", generator=g)).to(torch.bfloat16)[None].contiguous()
c = x[:, torch.randperm(N, device="cuda", generator=g)[:K]].contiguous()
ids, mind = ops.assign(x, c)
torch.cuda.synchronize()
t0 = time.time(); n = 0
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
while time.time() - t0 < 3:
    for _ in range(20): ops.assign(x, c, idx_out=ids, mind_out=mind)
    torch.cuda.synchronize(); n += 20
e.record(); torch.cuda.synchronize()
print(f"{s.elapsed_time(e)/n:.3f} ms/assign over {n} launches")
PY
kill $P
awk -F', ' -v tag=$1 '{gsub(" MHz","",$1); gsub(" W","",$2); if ($2 > 400) {n++; c+=$1; w+=$2}} END {if (n) printf "%s: %d samples under load, mean %.0f MHz, %.0f W\n", tag, n, c/n, w/n}' gpurun_out/clk_$1.csv
