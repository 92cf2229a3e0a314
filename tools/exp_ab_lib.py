"""A/B of two builds of libspidgpu.so on the same data (development aid).

SPIDGPU_LIB_PATH=... python tools/exp_ab_lib.py ell reps -> one line per build"""
import sys
import torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2103_01380_b200.configs import CONFIGS  # noqa: E402
from paper_2103_01380_b200.engine import Engine  # noqa: E402

ell = int(sys.argv[1]) if len(sys.argv) > 1 else 48
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
eng = Engine(0)
A = eng.generate(CONFIGS["cfg5"], 0, 64)
Y = eng.sketch(A, ell, seed=1)
torch.cuda.synchronize()
for trial in range(3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        eng.sketch(A, ell, seed=1, out=Y)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    print(f"ell={ell} trial {trial}: {ms:.3f} ms {A.numel() * 8 / ms / 1e9:.0f} TB/s*1e3", flush=True)
