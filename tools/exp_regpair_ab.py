"""Same-process A/B of the sketch-sized column ID over CTA pairs
(SPIDGPU_OPT_REG_PAIRS) vs one CTA per subdomain: config 3's 64 x (48 x 256)
fixed rank 32, and a tolerance-rule case, CUDA-event timed, interleaved.
python tools/exp_regpair_ab.py [rounds]"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2103_01380_b200 import _native as N  # noqa: E402
from paper_2103_01380_b200.engine import Engine  # noqa: E402
from paper_2103_01380_b200.spid import RankRule  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 5
eng = Engine(0)
torch.manual_seed(0)
cases = [("cfg3 64 x 48x256 fixed 32", torch.randn((64, 256, 48), dtype=torch.float64, device="cuda"),
          RankRule.fixed(32)),
         ("64 x 80x256 tol 1e-8", torch.randn((64, 256, 80), dtype=torch.float64, device="cuda"),
          RankRule.tolerance(1e-8)),
         ("64 x 64x200 fixed 40", torch.randn((64, 200, 64), dtype=torch.float64, device="cuda"),
          RankRule.fixed(40)),
         ("64 x 32x256 fixed 16", torch.randn((64, 256, 32), dtype=torch.float64, device="cuda"),
          RankRule.fixed(16)),
         ("128 x 48x256 fixed 32", torch.randn((128, 256, 48), dtype=torch.float64, device="cuda"),
          RankRule.fixed(32)),
         ("8 x 48x256 fixed 32", torch.randn((8, 256, 48), dtype=torch.float64, device="cuda"),
          RankRule.fixed(32))]
res = {}
for r in range(rounds):
    for pairs in (1, 0):
        eng.h.check(N.lib.spidgpu_set_option(eng.h.h, N.SPIDGPU_OPT_REG_PAIRS, pairs))
        for name, Y, rule in cases:
            eng.cpqr(Y, rule)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10):
                eng.cpqr(Y, rule)
            b.record()
            torch.cuda.synchronize()
            res.setdefault((name, pairs), []).append(a.elapsed_time(b) / 10 * 1e3)
for (name, pairs), v in sorted(res.items()):
    v = sorted(v)
    print(f"{name:28s} pairs={pairs}: min {v[0]:.1f} median {v[len(v) // 2]:.1f} us", flush=True)
