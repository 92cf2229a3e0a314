"""One performance-mode sketch of cfg3's 64 subdomains at a given ell (for ncu
captures of a single sketch_tc launch). python tools/exp_sketch_one.py ELL"""
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_2103_01380_b200.configs import CONFIGS  # noqa: E402
from paper_2103_01380_b200.engine import Engine  # noqa: E402

ell = int(sys.argv[1]) if len(sys.argv) > 1 else 48
eng = Engine(0)
A = eng.generate(CONFIGS["cfg3"], 0, 64)
Y = torch.empty((64, 256, ell), dtype=torch.float64, device="cuda")
for _ in range(2):
    eng.sketch(A, ell, seed=1, out=Y)
torch.cuda.synchronize()
print("ok", float(Y.abs().sum()))
