"""The pipeline's stage-2 column-ID shape (64 x (4096 x 128), tolerance 1e-5)
on random (full rank) and graded low-rank inputs, tall CTA pairs on and off,
CUDA-event timed. python tools/exp_stage2_shape.py"""
import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2103_01380_b200 import _native as N
from paper_2103_01380_b200.engine import Engine
from paper_2103_01380_b200.spid import RankRule
eng = Engine(0)
g = torch.Generator(device="cuda").manual_seed(1)
Yr = torch.randn((64, 128, 4096), dtype=torch.float64, device="cuda", generator=g)
U = torch.randn((64, 40, 4096), dtype=torch.float64, device="cuda", generator=g)
V = torch.randn((64, 128, 40), dtype=torch.float64, device="cuda", generator=g) * torch.logspace(0, -12, 40, dtype=torch.float64, device="cuda")
Yl = torch.bmm(V, U)
for name, Y in (("random", Yr), ("lowrank", Yl)):
    for pairs in (1, 0, 1, 0, 1, 0):
        eng.h.check(N.lib.spidgpu_set_option(eng.h.h, N.SPIDGPU_OPT_TALL_PAIRS, pairs))
        ts = []
        for _ in range(4):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); a.record()
            res = eng.cpqr(Y, RankRule.tolerance(1e-5))
            b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
        print(name, pairs, " ".join(f"{t:.2f}" for t in ts), "rank", int(res.rank.max()), flush=True)
