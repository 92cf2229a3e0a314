"""Pinned H2D bandwidth: one stream vs two concurrent streams, and H2D with a
concurrent D2H (full duplex) -- the e2e leg's transfer pattern."""
import torch

n = 2 << 30  # 2 GiB per buffer
h = [torch.empty(n // 8, dtype=torch.float64, pin_memory=True) for _ in range(2)]
d = [torch.empty(n // 8, dtype=torch.float64, device="cuda") for _ in range(2)]
st = [torch.cuda.Stream() for _ in range(2)]


def timed(fn, nbytes, reps=4):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    return reps * nbytes / (s.elapsed_time(e) / 1e3) / 1e9


def one():
    d[0].copy_(h[0], non_blocking=True)


def two():
    for i in range(2):
        with torch.cuda.stream(st[i]):
            d[i].copy_(h[i], non_blocking=True)


def duplex():
    with torch.cuda.stream(st[0]):
        d[0].copy_(h[0], non_blocking=True)
    with torch.cuda.stream(st[1]):
        h[1].copy_(d[1], non_blocking=True)


print(f"H2D one stream: {timed(one, n):.1f} GB/s")
print(f"H2D two streams: {timed(two, 2 * n):.1f} GB/s")
print(f"H2D + D2H concurrently: {timed(duplex, 2 * n):.1f} GB/s total")
