"""DMMA (explicit-Omega path) sketch timing on the config-3 batch with the Philox Omega routed
to it (SPIDGPU_OPT_DMMA_SKETCH). SPIDGPU_LIB_PATH=... python tools/exp_dmma_sketch.py"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2103_01380_b200 import _native as N  # noqa: E402
from paper_2103_01380_b200.configs import CONFIGS  # noqa: E402
from paper_2103_01380_b200.engine import Engine  # noqa: E402

eng = Engine(0)
A = eng.generate(CONFIGS["cfg5"], 0, 64)
eng.h.check(N.lib.spidgpu_set_option(eng.h.h, N.SPIDGPU_OPT_DMMA_SKETCH, 1))
Y = eng.sketch(A, 48, seed=1)
torch.cuda.synchronize()
best = 1e9
for _ in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        eng.sketch(A, 48, seed=1, out=Y)
    b.record()
    torch.cuda.synchronize()
    best = min(best, a.elapsed_time(b) / 3)
print(f"DMMA sketch ell 48, 64 x 163840x256: {best:.3f} ms", flush=True)
