"""Throughput of concurrent narrow tall column IDs (the pipeline's stage-1
shape, 64 x (4913 x 32), rank 16): K batches issued on K streams (one Engine
each) vs one after another, CUDA-event timed around the whole set.
python tools/exp_tall_concurrency.py"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2103_01380_b200.engine import Engine  # noqa: E402
from paper_2103_01380_b200.spid import RankRule  # noqa: E402

K = 4
engs = [Engine(0) for _ in range(K)]
streams = [torch.cuda.Stream() for _ in range(K)]
Ys = [torch.randn((64, 32, 4913), dtype=torch.float64, device="cuda") for _ in range(K)]
rule = RankRule.fixed(16)
for e, Y in zip(engs, Ys):
    e.cpqr(Y, rule)
torch.cuda.synchronize()


def timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    fn()
    torch.cuda.synchronize()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


for rep in range(3):
    for k in (1, 2, 4):
        def conc():
            cur = torch.cuda.current_stream()
            for i in range(k):
                streams[i].wait_stream(cur)
                with torch.cuda.stream(streams[i]):
                    engs[i].cpqr(Ys[i], rule, stream=streams[i])
            for i in range(k):
                cur.wait_stream(streams[i])

        def seq():
            for i in range(k):
                engs[0].cpqr(Ys[i], rule)
        print(f"k={k}: concurrent {timed(conc):.2f} ms, sequential {timed(seq):.2f} ms", flush=True)
