"""Time the ell = 80 sketch (config-3 batch) under the library named by SPIDGPU_LIB_PATH."""
import sys
import torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2103_01380_b200.configs import CONFIGS  # noqa: E402
from paper_2103_01380_b200.engine import Engine  # noqa: E402
ell = int(sys.argv[1]) if len(sys.argv) > 1 else 80
eng = Engine(0)
X = eng.generate(CONFIGS["cfg5"], 0, 64)
Y = eng.sketch(X, ell, seed=1)
torch.cuda.synchronize()
for trial in range(3):
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(5):
        eng.sketch(X, ell, seed=1, out=Y)
    s1.record()
    torch.cuda.synchronize()
    ms = s0.elapsed_time(s1) / 5
    print(f"ell={ell}: {ms:.3f} ms = {X.numel() * 8 / ms / 1e9:.0f} GB/s", flush=True)
