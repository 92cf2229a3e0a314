import sys, types, torch
sys.path.insert(0, "/root/repo")
import bench
from paper_2103_01380_b200.engine import Engine
cfg, field, first, count = bench.workload("cfg3", 0, 1)
eng = Engine(0)
A = eng.generate(field, first, count)
torch.cuda.synchronize()
for i in range(3):
    r = bench.pipeline_measure(cfg, A, types.SimpleNamespace())
    print(r['device_frames'], r['e2e']['value'], r['stage1_ms'], r['stage2_ms'], flush=True)
