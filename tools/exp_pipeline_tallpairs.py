"""Streaming pipeline (config-3 u field, device frames) with the tall
column-ID CTA pairs on and off (SPIDGPU_OPT_TALL_PAIRS on the cached handle),
interleaved: stage-1 / stage-2 device times and the archive bytes.
python tools/exp_pipeline_tallpairs.py [rounds]"""
import ctypes as C
import hashlib
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import bench  # noqa: E402
from paper_2103_01380_b200 import _native as N  # noqa: E402
from paper_2103_01380_b200 import pipeline as PL  # noqa: E402
from paper_2103_01380_b200.engine import Engine  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg, field_cfg, first, count = bench.workload("cfg3", 0, 1)
eng = Engine(0)
A = eng.generate(field_cfg, first, count)
field = bench.global_field(A, cfg.grid, cfg.block, qoi=1)
m, n = field.shape
frames = field.T
pc = PL.StreamConfig(dims=(cfg.grid,) * 3, blocks=(cfg.grid // cfg.block,) * 3, strides=(2, 2, 2), time_chunk=32,
                     stage1_rank=16, stage2_tol=1e-5, periodic=(1, 1, 1), qoi="u", provenance="bench")
h = N.handle(torch.cuda.current_device())
for r in range(rounds):
    for pairs in (1, 0):
        h.check(N.lib.spidgpu_set_option(h.h, N.SPIDGPU_OPT_TALL_PAIRS, pairs))
        torch.cuda.synchronize()
        with PL.Pipeline(pc) as p:
            t0 = time.perf_counter()
            for j in range(n):
                p.push(frames[j])
            nb = C.c_int64()
            p._check(N.lib.spidgpu_stream_finish(p.s, C.byref(nb)))
            t1 = time.perf_counter()
            view, ln = C.c_void_p(), C.c_int64()
            p.h.check(N.lib.spidgpu_archive_view(p.h.h, C.byref(view), C.byref(ln)))
            digest = hashlib.sha256(C.string_at(view.value, ln.value)).hexdigest()[:16]
            st = p.stats()
        print(f"pairs={pairs}: total {1e3 * (t1 - t0):.1f} ms; stage1 {st['stage1_ms']:.1f} stage2 {st['stage2_ms']:.1f}"
              f" ms; archive {digest}", flush=True)
