"""A/B the performance-mode sketch between the in-tree library and an
alternative build (SPIDGPU_LIB_PATH), alternating runs to cancel power-cap
drift. Usage: [SKETCH_AB_CONFIG=cfg2] python tools/exp_sketch_ab.py LIB_B [ell ...]"""
import os
import subprocess
import sys

CHILD = r'''
import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2103_01380_b200.configs import CONFIGS
from paper_2103_01380_b200.engine import Engine
import os
cfg = CONFIGS[os.environ.get("SKETCH_AB_CONFIG", "cfg3")]
eng = Engine(0); A = eng.generate(cfg, 0, 64)
st = torch.cuda.current_stream()
gb = A.numel() * 8 / 1e9
for ell in [int(x) for x in sys.argv[1:]]:
    Y = torch.empty((64, A.shape[1], ell), dtype=torch.float64, device="cuda")
    eng.sketch(A, ell, seed=1, out=Y); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    reps = int(os.environ.get("SKETCH_AB_REPS", "5"))
    for _ in range(reps): eng.sketch(A, ell, seed=1, out=Y)
    b.record(st); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    print(f"  ell {ell}: {ms:.3f} ms  {gb/ms:.2f} TB/s", flush=True)
'''

lib_b = sys.argv[1]
ells = sys.argv[2:] or ["48", "64"]
for rep in range(int(os.environ.get("SKETCH_AB_ROUNDS", "2"))):
    for name, lib in (("A", ""), ("B", lib_b)):
        env = dict(os.environ)
        if lib:
            env["SPIDGPU_LIB_PATH"] = os.path.abspath(lib)
        print(f"{name} rep {rep} {lib or 'in-tree'}", flush=True)
        subprocess.run([sys.executable, "-c", CHILD, *ells], env=env, check=True)
