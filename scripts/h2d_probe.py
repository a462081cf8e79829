import torch, time
x = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
y = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
for chunk in (1 << 24, 1 << 26, 1 << 28, 1 << 30):
    for _ in range(2): y.copy_(x, non_blocking=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for r in range(3):
        for o in range(0, 1 << 30, chunk):
            y[o:o + chunk].copy_(x[o:o + chunk], non_blocking=True)
    e.record(); torch.cuda.synchronize()
    print(f"H2D chunk {chunk >> 20} MiB: {3 * (1 << 30) / (s.elapsed_time(e) * 1e-3) / 1e9:.1f} GB/s")
