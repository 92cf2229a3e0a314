import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2103_01380_b200.configs import CONFIGS
from paper_2103_01380_b200.engine import Engine
cfg = CONFIGS['cfg3']; eng = Engine(0); A = eng.generate(CONFIGS['cfg5'], 0, 64)
st = torch.cuda.current_stream()
for ell in [16, 32, 48, 64, 48, 32]:
    Y = torch.empty((64, 256, ell), dtype=torch.float64, device='cuda')
    eng.sketch(A, ell, seed=1, out=Y); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(3): eng.sketch(A, ell, seed=1, out=Y)
    b.record(st); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    print(f"ell {ell}: {ms:.3f} ms  {21.47/ms:.2f} TB/s", flush=True)
