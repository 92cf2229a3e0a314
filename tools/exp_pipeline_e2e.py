"""Where the streaming pipeline's time goes: the push loop (device frames, or
one pinned host frame per call), spidgpu_stream_finish, and the copy of the
archive into Python bytes. python tools/exp_pipeline_e2e.py"""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
from paper_2103_01380_b200 import _native as N  # noqa: E402
from paper_2103_01380_b200 import pipeline as PL  # noqa: E402
from paper_2103_01380_b200.engine import Engine  # noqa: E402

cfg, field_cfg, first, count = bench.workload("cfg3", 0, 1)
eng = Engine(0)
A = eng.generate(field_cfg, first, count)
field = bench.global_field(A, cfg.grid, cfg.block, qoi=1)
m, n = field.shape
frames = field.T
host = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
host.copy_(frames)
hf = host.numpy()
pc = PL.StreamConfig(dims=(cfg.grid,) * 3, blocks=(cfg.grid // cfg.block,) * 3, strides=(2, 2, 2), time_chunk=32,
                     stage1_rank=16, stage2_tol=1e-5, periodic=(1, 1, 1), qoi="u", provenance="bench")
for src_name, src in (("device", frames), ("host", hf)) * 3:
    torch.cuda.synchronize()
    with PL.Pipeline(pc) as p:
        t0 = time.perf_counter()
        for j in range(n):
            p.push(src[j])
        t1 = time.perf_counter()
        nb = C.c_int64()
        p._check(N.lib.spidgpu_stream_finish(p.s, C.byref(nb)))
        t2 = time.perf_counter()
        view, ln = C.c_void_p(), C.c_int64()
        p.h.check(N.lib.spidgpu_archive_view(p.h.h, C.byref(view), C.byref(ln)))
        data = C.string_at(view.value, ln.value)
        t3 = time.perf_counter()
        st = p.stats()
    print(f"{src_name}: push loop {1e3 * (t1 - t0):.1f} ms, finish {1e3 * (t2 - t1):.1f} ms, bytes copy "
          f"{1e3 * (t3 - t2):.1f} ms, total {1e3 * (t2 - t0):.1f} ms; stage1 {st['stage1_ms']:.1f} "
          f"stage2 {st['stage2_ms']:.1f}", flush=True)
