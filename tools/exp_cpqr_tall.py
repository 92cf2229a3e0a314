"""Batched tall column ID (the archive's exact mode shape: 64 blocks of 4096
coarse rows x 256 snapshots, rank 32; and the pipeline's stage-1 shape, 4096 x
32, rank 16), timed with CUDA events. python tools/exp_cpqr_tall.py [reps]"""
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_2103_01380_b200.engine import Engine  # noqa: E402
from paper_2103_01380_b200.spid import RankRule  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
eng = Engine(0)
for rows, n, k in [(4096, 256, 32), (4096, 32, 16)]:
    Y = torch.randn((64, n, rows), dtype=torch.float64, device="cuda")
    eng.cpqr(Y, RankRule.fixed(k)).check()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        eng.cpqr(Y, RankRule.fixed(k))
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    print(f"64 x ({rows} x {n}) rank {k}: {ms:.3f} ms", flush=True)
