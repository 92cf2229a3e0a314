"""Stage breakdown (SPIDGPU_TRACE=1 CUDA-event marks on stderr) of the
archive compress/decompress legs of bench.py on config 3's u field.
python tools/exp_archive_trace.py"""
import os
import sys
import types

os.environ["SPIDGPU_TRACE"] = "1"
sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2103_01380_b200.engine import Engine  # noqa: E402

cfg, field, first, count = bench.workload("cfg3", 0, 1)
eng = Engine(0)
A = eng.generate(field, first, count)
torch.cuda.synchronize()
print(bench.archive_measure(cfg, A, types.SimpleNamespace()), flush=True)
print(bench.pipeline_measure(cfg, A, types.SimpleNamespace()), flush=True)
