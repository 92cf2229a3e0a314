"""Sketch duration inside the compress step vs back-to-back alone (config 3,
CUDA events on the launching stream). python tools/exp_sketch_context.py"""
import sys

import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
from paper_2103_01380_b200.engine import Engine, rule_for  # noqa: E402

cfg, field, first, count = bench.workload("cfg3", 0, 1)
eng = Engine(0)
A = eng.generate(field, first, count)
rule = rule_for(cfg)
res = eng.compress(A, cfg.ell, rule, seed=cfg.seed, want_sketch=True)
torch.cuda.synchronize()
st = torch.cuda.current_stream()


def run(mode, reps=20):
    ev = []
    for i in range(reps + 3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        eng.sketch(A, cfg.ell, seed=cfg.seed, out=res.sketch)
        b.record(st)
        if i >= 3:
            ev.append((a, b))
        if mode == "step":
            eng.h.check(bench._cpqr_into(eng, res, rule))
            eng.h.check(bench._gather_into(eng, A, res))
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in ev)
    return t[len(t) // 2], t[0], t[-1]


for mode in ["alone", "step", "alone", "step"]:
    med, lo, hi = run(mode)
    print(f"{mode:5s}: sketch median {med:.3f} ms (min {lo:.3f}, max {hi:.3f})", flush=True)
