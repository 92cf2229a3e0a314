"""Run the streaming two-stage compressor once warm and once
timed on the bench's u field (development aid / ncu target).

python tools/prof_pipeline.py
"""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import bench  # noqa: E402
from paper_2103_01380_b200 import pipeline as PL  # noqa: E402
from paper_2103_01380_b200.configs import CONFIGS  # noqa: E402
from paper_2103_01380_b200.engine import Engine  # noqa: E402

cfg = CONFIGS["cfg3"]
eng = Engine(0)
A = eng.generate(CONFIGS["cfg5"], 0, 64)
field = bench.global_field(A, cfg.grid, cfg.block, qoi=1)
m, n = field.shape
frames = field.T
pc = PL.StreamConfig(dims=(cfg.grid,) * 3, blocks=(cfg.grid // cfg.block,) * 3, strides=(2, 2, 2),
                     time_chunk=32, stage1_rank=16, stage2_tol=1e-5, periodic=(1, 1, 1), qoi="u",
                     provenance="bench")
for rep in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    with PL.Pipeline(pc) as p:
        for j in range(n):
            p.push(frames[j])
        data = p.finish()
        st = p.stats()
    torch.cuda.synchronize()
    print(f"rep {rep}: {1e3 * (time.perf_counter() - t):.1f} ms, archive {len(data)} B, stats {st}", flush=True)
