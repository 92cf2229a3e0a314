"""Batched register CPQR timing (development aid): the config-3 step's column
ID (64 subdomains, 48 x 256 sketches, fixed k = 32) and config 4's (216 x
80 x 256, blocked rule up to 64). SPIDGPU_LIB_PATH=... python tools/exp_cpqr_time.py"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2103_01380_b200.engine import Engine  # noqa: E402
from paper_2103_01380_b200.spid import RankRule  # noqa: E402

eng = Engine(0)
torch.manual_seed(0)
cases = [("cfg3 64 x 48x256 fixed 32", torch.randn((64, 256, 48), dtype=torch.float64, device="cuda"),
          RankRule.fixed(32)),
         ("cfg4 216 x 80x256 blocked 64/8/1e-3",
          torch.randn((216, 256, 80), dtype=torch.float64, device="cuda"), RankRule.blocked(64, 8, 1e-3))]
for name, Y, rule in cases:
    ref = eng.cpqr(Y, rule)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            eng.cpqr(Y, rule)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 10)
    print(f"{name}: {1e3 * best:.1f} us, ranks {int(ref.rank.min())}..{int(ref.rank.max())}, "
          f"idx sum {int(ref.indices.sum())}", flush=True)
