"""Device-resident archive compress (sketch mode) of the config-3 u field, as
bench.py's archive leg runs it: wall time per call and (under ncu) the kernels.
python tools/exp_archive_one.py [reps]"""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import bench  # noqa: E402
from paper_2103_01380_b200 import _native as N  # noqa: E402
from paper_2103_01380_b200.engine import Engine  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg, field_cfg, first, count = bench.workload("cfg3", 0, 1)
eng = Engine(0)
A = eng.generate(field_cfg, first, count)
field = bench.global_field(A, cfg.grid, cfg.block, qoi=1)
m, n = field.shape
h = N.handle(torch.cuda.current_device())
rr = N.RankRule(N.RULE_FIXED, 0, cfg.k, 0, 0.0)
nb = C.c_int64()
spec = N.archive_spec((cfg.grid,) * 3, (cfg.grid // cfg.block,) * 3, (2,) * 3, (1, 1, 1), N.ARCHIVE_SKETCH,
                      cfg.k + cfg.p, cfg.seed, "u", "bench")
for i in range(reps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    h.check(N.lib.spidgpu_archive_compress(h.h, C.c_void_p(field.data_ptr()), m, n, m, 1, C.byref(spec),
                                           C.byref(rr), C.byref(nb)))
    torch.cuda.synchronize()
    print(f"archive compress (device input): {1e3 * (time.perf_counter() - t):.2f} ms, {nb.value} bytes",
          flush=True)
