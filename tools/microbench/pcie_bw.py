"""Pinned host<->device copy bandwidth (the bound of bench.py's e2e leg)."""
import torch

n = 2 << 30  # 2 GiB
h = torch.empty(n // 8, dtype=torch.float64, pin_memory=True)
d = torch.empty(n // 8, dtype=torch.float64, device="cuda")
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in (("H2D", lambda: d.copy_(h, non_blocking=True)),
                 ("D2H", lambda: h.copy_(d, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(5):
        fn()
    e.record()
    torch.cuda.synchronize()
    print(f"{name} {5 * n / (s.elapsed_time(e) / 1e3) / 1e9:.1f} GB/s")
