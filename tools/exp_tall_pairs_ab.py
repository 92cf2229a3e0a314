"""Same-process A/B of the tall column ID over CTA pairs (SPIDGPU_OPT_TALL_PAIRS)
vs one CTA per block: the batched 64 x (4096 x 256) rank-32 column ID and the
exact-mode archive compress of the config-3 u field (device input), CUDA-event
timed, interleaved. python tools/exp_tall_pairs_ab.py [rounds]"""
import ctypes as C
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import bench  # noqa: E402
from paper_2103_01380_b200 import _native as N  # noqa: E402
from paper_2103_01380_b200.engine import Engine  # noqa: E402
from paper_2103_01380_b200.spid import RankRule  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 5
eng = Engine(0)
h = N.handle(torch.cuda.current_device())
Y = torch.randn((64, 256, 4096), dtype=torch.float64, device="cuda")
cfg, field_cfg, first, count = bench.workload("cfg3", 0, 1)
A = eng.generate(field_cfg, first, count)
field = bench.global_field(A, cfg.grid, cfg.block, qoi=1)
m, n = field.shape
rr = N.RankRule(N.RULE_FIXED, 0, cfg.k, 0, 0.0)
nb = C.c_int64()
spec = N.archive_spec((cfg.grid,) * 3, (cfg.grid // cfg.block,) * 3, (2,) * 3, (1, 1, 1), N.ARCHIVE_EXACT,
                      0, cfg.seed, "u", "bench")


def timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def cpqr():
    eng.cpqr(Y, RankRule.fixed(32))


def archive():
    h.check(N.lib.spidgpu_archive_compress(h.h, C.c_void_p(field.data_ptr()), m, n, m, 1, C.byref(spec),
                                           C.byref(rr), C.byref(nb)))


res = {}
for r in range(rounds):
    for pairs in (1, 0):
        for hh in (h, eng.h):
            hh.check(N.lib.spidgpu_set_option(hh.h, N.SPIDGPU_OPT_TALL_PAIRS, pairs))
        for name, fn in (("cpqr 64x(4096x256) k32", cpqr), ("archive exact cfg3 u", archive)):
            fn()
            res.setdefault((name, pairs), []).append(timed(fn))
for (name, pairs), v in sorted(res.items()):
    v = sorted(v)
    print(f"{name:26s} pairs={pairs}: min {v[0]:.2f} median {v[len(v) // 2]:.2f} ms ({nb.value} bytes)", flush=True)
