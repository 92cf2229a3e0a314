"""A/B the verify kernel between the in-tree library and an alternative build
(SPIDGPU_LIB_PATH) on config 3. python tools/exp_verify_ab.py LIB_B"""
import os
import subprocess
import sys

CHILD = r'''
import sys, torch
sys.path.insert(0, "/root/repo")
import bench
from paper_2103_01380_b200.engine import Engine, rule_for
cfg, field, first, count = bench.workload("cfg3", 0, 1)
eng = Engine(0); A = eng.generate(field, first, count)
res = eng.compress(A, cfg.ell, rule_for(cfg), seed=cfg.seed)
eng.verify(A, res); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5): eng.verify(A, res)
b.record(); torch.cuda.synchronize()
print(f"  verify {a.elapsed_time(b) / 5:.3f} ms", flush=True)
'''
for rep in range(2):
    for name, lib in (("A", ""), ("B", sys.argv[1])):
        env = dict(os.environ)
        if lib:
            env["SPIDGPU_LIB_PATH"] = os.path.abspath(lib)
        print(f"{name} rep {rep} {lib or 'in-tree'}", flush=True)
        subprocess.run([sys.executable, "-c", CHILD], env=env, check=True)
