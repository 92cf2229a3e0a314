"""Time the archive path on the GPU (device-resident field, synchronous ABI
calls, wall clock around each call after warm-up).

    python tools/archive_time.py [--grid 256] [--n 32] [--blocks 4] [--stride 2] [--rank 8]
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_01380_b200 import archive as A  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--blocks", type=int, default=4)
    ap.add_argument("--stride", type=int, default=2)
    ap.add_argument("--rank", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--modes", default="sketch,exact")
    a = ap.parse_args()
    g, n = a.grid, a.n
    m = g ** 3
    x = torch.linspace(0, 2 * torch.pi, g + 1, device="cuda", dtype=torch.float64)[:-1]
    X, Y, Z = torch.meshgrid(x, x, x, indexing="ij")
    t = torch.linspace(0, 1, n, device="cuda", dtype=torch.float64)
    f = torch.empty((n, m), device="cuda", dtype=torch.float64)
    for j in range(n):
        f[j] = (torch.sin(X + t[j]) * torch.cos(Y) * torch.cos(Z) +
                0.3 * torch.cos(2 * X) * torch.sin(Y + Z - t[j])).permute(2, 1, 0).reshape(-1)
    f += 1e-6 * torch.randn_like(f)
    field = f.T  # m x n column-major view
    res = {"grid": g, "n": n, "blocks": a.blocks ** 3, "stride": a.stride, "rank": a.rank,
           "field_gb": m * n * 8 / 1e9}
    dims, blocks, strides = (g,) * 3, (a.blocks,) * 3, (a.stride,) * 3
    # CRC throughput over the field bytes (device buffer)
    raw = field.T.contiguous().view(torch.uint8).reshape(-1)
    s = timed(lambda: A.crc32(raw), a.reps)
    res["crc32_gbps"] = raw.numel() / s / 1e9
    for mode in a.modes.split(","):
        kw = dict(mode=A.ARCHIVE_SKETCH, ell=a.rank + 8, seed=1) if mode == "sketch" else {}
        data = None

        def run():
            nonlocal data
            data = A.compress_field(field, dims, blocks, strides, periodic=(1, 1, 1), rank=a.rank, **kw)
        s = timed(run, a.reps)
        out = torch.empty((n, m), device="cuda", dtype=torch.float64).T
        sd = timed(lambda: A.decompress(data, out=out), a.reps)
        err = (torch.linalg.norm(out - field) / torch.linalg.norm(field)).item()
        res[mode] = {"compress_s": s, "compress_gbps": m * n * 8 / s / 1e9, "archive_mb": len(data) / 1e6,
                     "cf": m * n * 8 / len(data), "decompress_s": sd, "decompress_gbps": m * n * 8 / sd / 1e9,
                     "rel_err": err}
    print(json.dumps(res))




def phases(grid=256, n=32, blocks=4, stride=2, rank=8):
    """Split compress_field into the ABI call, the fetch and the bytes copy."""
    import ctypes as C
    from paper_2103_01380_b200 import _native as N
    import numpy as np
    m = grid ** 3
    field = torch.randn((n, m), device="cuda", dtype=torch.float64).T
    for mode in (A.ARCHIVE_SKETCH, A.ARCHIVE_EXACT):
        spec = N.archive_spec((grid,) * 3, (blocks,) * 3, (stride,) * 3, (1, 1, 1), mode, rank + 8, 1)
        rr = N.RankRule(N.RULE_FIXED, 0, rank, 0, 0.0)
        h = N.handle(0)
        nb = C.c_int64()
        call = lambda: h.check(N.lib.spidgpu_archive_compress(h.h, C.c_void_p(field.data_ptr()), m, n, m, 1,  # noqa: E731
                                                              C.byref(spec), C.byref(rr), C.byref(nb)))
        s_call = timed(call, 3)
        out = np.empty(nb.value, dtype=np.uint8)
        s_fetch = timed(lambda: N.lib.spidgpu_archive_fetch(h.h, C.c_void_p(out.ctypes.data), nb.value), 3)
        s_bytes = timed(lambda: out.tobytes(), 3)
        print(json.dumps({"mode": mode, "call_s": s_call, "fetch_s": s_fetch, "tobytes_s": s_bytes,
                          "archive_mb": nb.value / 1e6}))


if __name__ == "__main__":
    if "--phases" in sys.argv:
        phases()
    else:
        main()
