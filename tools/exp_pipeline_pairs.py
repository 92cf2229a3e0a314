import ctypes as C, sys, time, torch
sys.path.insert(0, "/root/repo")
import bench
from paper_2103_01380_b200 import _native as N
from paper_2103_01380_b200 import pipeline as PL
from paper_2103_01380_b200.engine import Engine
cfg, field_cfg, first, count = bench.workload("cfg3", 0, 1)
eng = Engine(0)
A = eng.generate(field_cfg, first, count)
field = bench.global_field(A, cfg.grid, cfg.block, qoi=1)
m, n = field.shape
frames = field.T
pc = PL.StreamConfig(dims=(cfg.grid,) * 3, blocks=(cfg.grid // cfg.block,) * 3, strides=(2, 2, 2), time_chunk=32,
                     stage1_rank=16, stage2_tol=1e-5, periodic=(1, 1, 1), qoi="u", provenance="bench")
for rep in range(3):
    for pairs in (1, 0):
        torch.cuda.synchronize()
        with PL.Pipeline(pc) as p:
            p.h.check(N.lib.spidgpu_set_option(p.h.h, N.SPIDGPU_OPT_TALL_PAIRS, pairs))
            t0 = time.perf_counter()
            for j in range(n):
                p.push(frames[j])
            nb = C.c_int64()
            p._check(N.lib.spidgpu_stream_finish(p.s, C.byref(nb)))
            t1 = time.perf_counter()
            st = p.stats()
        print(f"pairs {pairs}: device frames {1e3*(t1-t0):.1f} ms, stage1 {st['stage1_ms']:.1f} stage2 {st['stage2_ms']:.1f}", flush=True)
