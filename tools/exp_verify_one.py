"""One config-3 compress + verify (64 subdomains), for ncu captures of a single
verify_tma_kernel launch. python tools/exp_verify_one.py"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import bench  # noqa: E402
from paper_2103_01380_b200.engine import Engine, rule_for  # noqa: E402

cfg, field, first, count = bench.workload("cfg3", 0, 1)
eng = Engine(0)
A = eng.generate(field, first, count)
res = eng.compress(A, cfg.ell, rule_for(cfg), seed=cfg.seed)
e2, r2 = eng.verify(A, res)
torch.cuda.synchronize()
print("ok", float((e2.sum() / r2.sum()).sqrt()))
