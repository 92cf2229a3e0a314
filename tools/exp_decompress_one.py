"""Archive compress (sketch mode) then decompress of the config-3 u field; times the
decompress (wall) and, under ncu, lists its kernels. python tools/exp_decompress_one.py [reps]"""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import bench  # noqa: E402
from paper_2103_01380_b200 import archive as AR  # noqa: E402
from paper_2103_01380_b200.engine import Engine  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg, field_cfg, first, count = bench.workload("cfg3", 0, 1)
eng = Engine(0)
A = eng.generate(field_cfg, first, count)
field = bench.global_field(A, cfg.grid, cfg.block, qoi=1)
m, n = field.shape
data = AR.compress_field(field, (cfg.grid,) * 3, (cfg.grid // cfg.block,) * 3, (2,) * 3, periodic=(1, 1, 1),
                         rank=cfg.k, mode=AR.ARCHIVE_SKETCH, ell=cfg.k + cfg.p, seed=cfg.seed)
dec = torch.empty((n, m), dtype=torch.float64, device="cuda").T
for _ in range(reps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    AR.decompress(data, out=dec)
    torch.cuda.synchronize()
    print(f"decompress: {1e3 * (time.perf_counter() - t):.2f} ms", flush=True)
