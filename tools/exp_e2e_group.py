"""compress_host (pinned host in/out, 2 lanes) on config 3's 64 subdomains for several
group sizes: GB/s of raw field. python tools/exp_e2e_group.py"""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import bench  # noqa: E402
from paper_2103_01380_b200.engine import Engine, rule_for  # noqa: E402

cfg, field, first, count = bench.workload("cfg3", 0, 1)
eng = Engine(0)
A = eng.generate(field, first, count)
rule = rule_for(cfg)
kcap = rule.cap(cfg.ell, cfg.n)
ne = count
a_host = torch.empty((ne,) + tuple(A.shape[1:]), dtype=torch.float64, pin_memory=True)
a_host.copy_(A[:ne])
out = {"indices": torch.empty((ne, kcap), dtype=torch.int64, pin_memory=True),
       "coeffs": torch.empty((ne, cfg.n, kcap), dtype=torch.float64, pin_memory=True),
       "skel": torch.empty((ne, kcap, cfg.m), dtype=torch.float64, pin_memory=True),
       "rank": torch.empty(ne, dtype=torch.int64, pin_memory=True),
       "residual_fro": torch.empty(ne, dtype=torch.float64, pin_memory=True),
       "status": torch.empty(ne, dtype=torch.int32, pin_memory=True)}
for g in (2, 4, 8, 16, 4, 8):
    eng.compress_host(a_host, cfg.ell, rule, seed=cfg.seed, subdomain_base=first, group=g, out=out)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        eng.compress_host(a_host, cfg.ell, rule, seed=cfg.seed, subdomain_base=first, group=g, out=out)
    sec = (time.perf_counter() - t) / 3
    print(f"group {g}: {1e3 * sec:.1f} ms, {cfg.raw_bytes(ne) / sec / 1e9:.2f} GB/s", flush=True)
