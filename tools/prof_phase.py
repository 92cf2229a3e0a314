"""Run one phase of the compress path a few times (for ncu captures).

python tools/prof_phase.py <sketch|cpqr|gather|verify|compress> [cfg] [reps]
"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2103_01380_b200.configs import CONFIGS  # noqa: E402
from paper_2103_01380_b200.engine import Engine, rule_for  # noqa: E402


def main():
    phase = sys.argv[1]
    name = sys.argv[2] if len(sys.argv) > 2 else "cfg3"
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    cfg = CONFIGS[name]
    S = cfg.per_gpu_subdomains or cfg.subdomains
    gen = CONFIGS["cfg5"] if cfg.per_gpu_subdomains else cfg
    eng = Engine(0)
    A = eng.generate(gen, 0, S)
    rule = rule_for(cfg)
    r = eng.compress(A, cfg.ell, rule, seed=cfg.seed, want_sketch=True)
    r.check()
    for _ in range(reps):
        if phase == "sketch":
            eng.sketch(A, cfg.ell, seed=cfg.seed, out=r.sketch)
        elif phase == "cpqr":
            eng.cpqr(r.sketch, rule)
        elif phase == "gather":
            eng.gather(A, r)
        elif phase == "verify":
            eng.verify(A, r)
        else:
            eng.compress(A, cfg.ell, rule, seed=cfg.seed, out=r)
    torch.cuda.synchronize()
    print("ok", phase, name, reps)


if __name__ == "__main__":
    main()
