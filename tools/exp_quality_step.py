"""The bench's quality_spid timed step alone (ell = 80 compress with the blocked rule + coarse
gather), config 3's 64 subdomains. SPIDGPU_LIB_PATH=... python tools/exp_quality_step.py"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import bench  # noqa: E402
from paper_2103_01380_b200.engine import Engine  # noqa: E402
from paper_2103_01380_b200.spid import RankRule  # noqa: E402

cfg, field, first, count = bench.workload("cfg3", 0, 1)
eng = Engine(0)
A = eng.generate(field, first, count)
rule = RankRule.blocked(64, 2, 3e-4)
spec = eng.block_spec(field, 2)
r = eng.compress(A, 64 + cfg.p, rule, seed=cfg.seed, want_skel=False)
eng.gather_coarse(A, r, spec)
torch.cuda.synchronize()
best = 1e9
for _ in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        eng.compress(A, 64 + cfg.p, rule, seed=cfg.seed, want_skel=False, out=r)
        eng.gather_coarse(A, r, spec)
    b.record()
    torch.cuda.synchronize()
    best = min(best, a.elapsed_time(b) / 5)
print(f"quality step: {best:.3f} ms", flush=True)
