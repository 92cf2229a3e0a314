"""Does overlapping group g's CPQR + skeleton gather (second stream) with group
g+1's sketch (first stream, persistent grid capped to leave SMs free) shorten
the config-3 compress step? python tools/exp_overlap.py"""
import ctypes as C
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_2103_01380_b200 import _native as N  # noqa: E402
from paper_2103_01380_b200.configs import CONFIGS  # noqa: E402
from paper_2103_01380_b200.engine import Engine, rule_for  # noqa: E402

cfg = CONFIGS["cfg3"]
eng = Engine(0)
A = eng.generate(CONFIGS["cfg5"], 0, 64)
rule = rule_for(cfg)
res = eng.compress(A, cfg.ell, rule, seed=cfg.seed, want_sketch=True)
torch.cuda.synchronize()
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
S, n, m = A.shape
kc = res.kcap
sA = torch.cuda.Stream()
sB = torch.cuda.Stream()


def cpqr_gather(g0, g1, st):
    Y = res.sketch[g0:g1]
    ell = Y.shape[2]
    eng.h.check(N.lib.spidgpu_cpqr_id_batched(
        eng.h.h, p(Y), ell, n, ell, ell * n, g1 - g0, C.byref(rule.c()), kc, p(res.indices[g0:g1]),
        p(res.coeffs[g0:g1]), kc * n, p(res.rank[g0:g1]), p(res.residual_fro[g0:g1]),
        p(res.status[g0:g1]), None, None, None, C.c_void_p(st.cuda_stream)))
    eng.h.check(N.lib.spidgpu_gather_batched(eng.h.h, p(A[g0:g1]), m, n, m, m * n, g1 - g0,
                                             p(res.indices[g0:g1]), kc, p(res.rank[g0:g1]),
                                             p(res.skel[g0:g1]), m, m * kc, C.c_void_p(st.cuda_stream)))


def step(G):
    bounds = [S * i // G for i in range(G + 1)]
    cur = torch.cuda.current_stream()
    sA.wait_stream(cur)
    sB.wait_stream(cur)
    for i in range(G):
        g0, g1 = bounds[i], bounds[i + 1]
        eng.sketch(A[g0:g1], cfg.ell, seed=cfg.seed, subdomain_base=g0, out=res.sketch[g0:g1], stream=sA)
        ev = torch.cuda.Event()
        ev.record(sA)
        sB.wait_event(ev)
        cpqr_gather(g0, g1, sB)
    cur.wait_stream(sA)
    cur.wait_stream(sB)


ref_idx = res.indices.clone()
for sms in [0, 140, 132, 120]:
    N.lib.spidgpu_set_option(eng.h.h, N.SPIDGPU_OPT_SKETCH_SMS, sms)
    for G in [1, 2, 4, 8]:
        for _ in range(2):
            step(G)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            step(G)
        b.record()
        torch.cuda.synchronize()
        ok = torch.equal(res.indices, ref_idx)
        print(f"sketch_sms {sms or 148:3d} groups {G}: {a.elapsed_time(b) / 5:.3f} ms/step  same={ok}",
              flush=True)
N.lib.spidgpu_set_option(eng.h.h, N.SPIDGPU_OPT_SKETCH_SMS, 0)
