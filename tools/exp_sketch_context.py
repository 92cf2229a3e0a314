import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2103_01380_b200.configs import CONFIGS
from paper_2103_01380_b200.engine import Engine, rule_for
cfg = CONFIGS['cfg3']; big = CONFIGS['cfg5']
eng = Engine(0); A = eng.generate(big, 0, 64); rule = rule_for(cfg)
r = eng.compress(A, cfg.ell, rule, seed=cfg.seed, want_sketch=True); r.check()
st = torch.cuda.current_stream()
def ev(): return torch.cuda.Event(enable_timing=True)
def run(mode, reps=6):
    ts = []
    for i in range(reps):
        if mode == 'after_gather': eng.gather(A, r)
        if mode == 'after_cpqr': eng.cpqr(r.sketch, rule)
        if mode == 'after_flush':
            buf = torch.empty(256 * 2**20, dtype=torch.uint8, device='cuda'); buf.fill_(1)
        a, b = ev(), ev(); a.record(st)
        eng.sketch(A, cfg.ell, seed=cfg.seed, out=r.sketch)
        b.record(st); ts.append((a, b))
    torch.cuda.synchronize()
    v = [x.elapsed_time(y) for x, y in ts][1:]
    print(mode, ['%.3f' % t for t in v])
for m in ['alone', 'after_gather', 'after_cpqr', 'after_flush', 'alone']: run(m)
