"""ell = 80 single-pass (slice-split CTA pair) check and timing (development aid).

python tools/exp_sketch80.py -- bitwise batch independence, the bound vs the
two-pass DMMA reference, and event timings at config 4's shape."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2103_01380_b200 import spid  # noqa: E402
from paper_2103_01380_b200 import _native as N  # noqa: E402
from paper_2103_01380_b200.configs import CONFIGS  # noqa: E402
from paper_2103_01380_b200.engine import Engine  # noqa: E402

eng = Engine(0)
torch.manual_seed(0)
A = torch.randn((3, 256, 9000), dtype=torch.float64, device="cuda")
y = eng.sketch(A, 80, seed=4)
torch.cuda.synchronize()
import oracle  # noqa: E402
o = oracle.port()
for s in range(3):
    om = spid.philox_omega(4, s, 80, 9000)
    a = np.asfortranarray(A[s].cpu().numpy().T)
    yr = o.matmul(om, a)
    yy = np.asfortranarray(y[s].cpu().numpy().T)
    B = np.abs(om) @ np.abs(a)
    print("subdomain", s, "max |dy|/B", float(np.max(np.abs(yy - yr) / B)), flush=True)
y1 = eng.sketch(A[1:2].contiguous(), 80, seed=4, subdomain_base=1)
print("batch independent:", bool(torch.equal(y1, y[1:2])), flush=True)
cfg = CONFIGS["cfg4"]
X = eng.generate(CONFIGS["cfg5"], 0, 64)
Y = eng.sketch(X, 80, seed=1)
torch.cuda.synchronize()
for trial in range(3):
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(5):
        eng.sketch(X, 80, seed=1, out=Y)
    s1.record()
    torch.cuda.synchronize()
    ms = s0.elapsed_time(s1) / 5
    print(f"ell=80 64 x 163840x256: {ms:.3f} ms = {X.numel() * 8 / ms / 1e9:.0f} GB/s", flush=True)
