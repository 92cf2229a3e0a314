"""Sketch time per ell, interleaved in one process (development aid):
SPIDGPU_LIB_PATH=... python tools/exp_ell_matrix.py [ell[:pairs] ...] -> min / median ms per
entry (pairs = SPIDGPU_OPT_SKETCH_PAIRS for that entry, default 1)."""
import statistics
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2103_01380_b200.configs import CONFIGS  # noqa: E402
from paper_2103_01380_b200.engine import Engine  # noqa: E402

from paper_2103_01380_b200 import _native as N  # noqa: E402

ells = sys.argv[1:] or ["48", "64", "80"]
eng = Engine(0)
A = eng.generate(CONFIGS["cfg5"], 0, 64)


def run(key, out=None):
    ell, _, pm = key.partition(":")
    eng.h.check(N.lib.spidgpu_set_option(eng.h.h, N.SPIDGPU_OPT_SKETCH_PAIRS, int(pm or 1)))
    return eng.sketch(A, int(ell), seed=1, out=out)


Ys = {e: run(e) for e in ells}
torch.cuda.synchronize()
t = {e: [] for e in ells}
for rnd in range(6):
    for e in ells:
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        run(e, Ys[e])
        s0.record()
        for _ in range(4):
            run(e, Ys[e])
        s1.record()
        torch.cuda.synchronize()
        t[e].append(s0.elapsed_time(s1) / 4)
for e in ells:
    print(f"ell={e}: min {min(t[e]):.3f} med {statistics.median(t[e]):.3f} ms "
          f"({A.numel() * 8 / min(t[e]) / 1e9:.2f} TB/s best)", flush=True)
