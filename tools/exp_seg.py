"""Sketch segment-length / data-dependence experiment (development aid).

python tools/exp_seg.py  -- times the tcgen05 sketch on the config-3 batch and
on N(0,1) data of the same shape for several segment lengths, with the
converter-warp flush counts by cause (spidgpu_debug_counters)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2103_01380_b200 import _native as N  # noqa: E402
from paper_2103_01380_b200.configs import CONFIGS  # noqa: E402
from paper_2103_01380_b200.engine import Engine  # noqa: E402


def main():
    eng = Engine(0)
    cfg = CONFIGS["cfg3"]
    big = CONFIGS["cfg5"]
    ell = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.ell
    A = eng.generate(big, 0, 64)
    torch.cuda.synchronize()
    R = torch.randn_like(A[:1]).expand_as(A).contiguous() if False else None
    cnt = (C.c_int64 * 3)()
    for name, X in (("cfg3", A), ("randn", None)):
        if X is None:
            A.normal_()
            X = A
        for seg in (4096, 8192, 16384, 65536):
            eng.h.check(N.lib.spidgpu_set_option(eng.h.h, N.SPIDGPU_OPT_SKETCH_SEG_ROWS, seg))
            Y = eng.sketch(X, ell, seed=cfg.seed)
            torch.cuda.synchronize()
            eng.h.check(N.lib.spidgpu_debug_counters(eng.h.h, cnt, 3, 1))
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            s.record()
            for _ in range(reps):
                eng.sketch(X, ell, seed=cfg.seed, out=Y)
            e.record()
            torch.cuda.synchronize()
            ms = s.elapsed_time(e) / reps
            eng.h.check(N.lib.spidgpu_debug_counters(eng.h.h, cnt, 3, 1))
            print(f"{name} ell={ell} seg={seg}: {ms:.3f} ms  {X.numel() * 8 / ms / 1e9:.0f} GB/s  "
                  f"flushes/launch seg={cnt[0] / reps:.0f} overflow={cnt[1] / reps:.0f} "
                  f"fallback={cnt[2] / reps:.0f}", flush=True)
    eng.h.check(N.lib.spidgpu_set_option(eng.h.h, N.SPIDGPU_OPT_SKETCH_SEG_ROWS, 0))


if __name__ == "__main__":
    main()
