"""Per-phase timing of the compress path on one GPU (development aid).

python tools/quick_time.py [cfg3|cfg2|cfg1|cfg4] [reps]
"""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2103_01380_b200.configs import CONFIGS  # noqa: E402
from paper_2103_01380_b200.engine import Engine, rule_for  # noqa: E402


def ev_time(fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    cfg = CONFIGS[name]
    if cfg.per_gpu_subdomains:
        big = CONFIGS["cfg5"]
        S = cfg.per_gpu_subdomains
        gen_cfg = big
    else:
        S = cfg.subdomains
        gen_cfg = cfg
    eng = Engine(0)
    t0 = time.time()
    A = eng.generate(gen_cfg, 0, S)
    torch.cuda.synchronize()
    print(f"{name}: S={S} m={cfg.m} n={cfg.n} ell={cfg.ell} k={cfg.k}  A={A.numel()*8/1e9:.2f} GB"
          f"  gen {time.time()-t0:.2f}s", flush=True)
    rule = rule_for(cfg)
    r = eng.compress(A, cfg.ell, rule, seed=cfg.seed, want_sketch=True)
    r.check()
    Y = r.sketch
    flops = 2.0 * cfg.ell * cfg.m * cfg.n * S
    bytes_a = 8.0 * cfg.m * cfg.n * S
    t_sk = ev_time(lambda: eng.sketch(A, cfg.ell, seed=cfg.seed, out=Y), reps)
    print(f"sketch   {t_sk:8.3f} ms  {flops/t_sk/1e9:7.2f} TFLOP/s  {bytes_a/t_sk/1e6:8.1f} GB/s", flush=True)
    t_qr = ev_time(lambda: eng.cpqr(Y, rule), reps)
    print(f"cpqr     {t_qr:8.3f} ms", flush=True)
    t_g = ev_time(lambda: eng.gather(A, r), reps)
    gb = 2.0 * 8 * cfg.m * cfg.k * S
    print(f"gather   {t_g:8.3f} ms  {gb/t_g/1e6:8.1f} GB/s", flush=True)
    t_c = ev_time(lambda: eng.compress(A, cfg.ell, rule, seed=cfg.seed, out=r), reps)
    print(f"compress {t_c:8.3f} ms  raw {bytes_a/t_c/1e6:8.1f} GB/s", flush=True)
    t_v = ev_time(lambda: eng.verify(A, r), reps)
    vfl = 2.0 * cfg.k * cfg.m * cfg.n * S
    print(f"verify   {t_v:8.3f} ms  {vfl/t_v/1e9:7.2f} TFLOP/s  {bytes_a/t_v/1e6:8.1f} GB/s", flush=True)
    e2, r2 = eng.verify(A, r)
    ranks = r.rank.cpu()
    print("rel err", (e2.sum() / r2.sum()).sqrt().item(), "ranks", ranks.min().item(), ranks.max().item(),
          "CF", (cfg.m * cfg.n * S) / (ranks.sum().item() * (cfg.m + cfg.n)))


if __name__ == "__main__":
    main()
