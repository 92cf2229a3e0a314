"""Sustained (power-capped) A/B of the tcgen05 sketch's CTA-pair mode on
config 3: blocks of 30 back-to-back sketches, alternating modes.
python tools/exp_sketch_pairs_sustained.py"""
import sys

import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
from paper_2103_01380_b200 import _native as N  # noqa: E402
from paper_2103_01380_b200.engine import Engine  # noqa: E402

cfg, field, first, count = bench.workload("cfg3", 0, 1)
eng = Engine(0)
A = eng.generate(field, first, count)
Y = torch.empty((count, cfg.n, cfg.ell), dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
for rnd in range(3):
    for mode in (1, 2):
        N.lib.spidgpu_set_option(eng.h.h, N.SPIDGPU_OPT_SKETCH_PAIRS, mode)
        eng.sketch(A, cfg.ell, seed=cfg.seed, out=Y)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(30):
            eng.sketch(A, cfg.ell, seed=cfg.seed, out=Y)
        b.record(st)
        torch.cuda.synchronize()
        print(f"round {rnd} {'pairs' if mode == 2 else 'single'}: {a.elapsed_time(b) / 30:.3f} ms", flush=True)
N.lib.spidgpu_set_option(eng.h.h, N.SPIDGPU_OPT_SKETCH_PAIRS, 1)
