"""Development aid: sketch kernel time vs GPU / HBM temperature and power.

python tools/exp_sketch_thermal.py
"""
import sys
import time

import pynvml
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2103_01380_b200.configs import CONFIGS  # noqa: E402
from paper_2103_01380_b200.engine import Engine, rule_for  # noqa: E402

pynvml.nvmlInit()
hd = pynvml.nvmlDeviceGetHandleByIndex(0)


def state():
    t = pynvml.nvmlDeviceGetTemperature(hd, pynvml.NVML_TEMPERATURE_GPU)
    try:
        mt = pynvml.nvmlDeviceGetFieldValues(hd, [pynvml.NVML_FI_DEV_MEMORY_TEMP])[0].value.uiVal
    except Exception:
        mt = -1
    p = pynvml.nvmlDeviceGetPowerUsage(hd) / 1000
    mc = pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_MEM)
    sc = pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM)
    return f"gpuT={t} memT={mt} P={p:.0f}W smclk={sc} memclk={mc}"


cfg = CONFIGS["cfg3"]
eng = Engine(0)
A = eng.generate(CONFIGS["cfg5"], 0, 64)
r = eng.compress(A, cfg.ell, rule_for(cfg), seed=cfg.seed, want_sketch=True)
st = torch.cuda.current_stream()


def burst(n):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in ev:
        a.record(st)
        eng.sketch(A, cfg.ell, seed=cfg.seed, out=r.sketch)
        b.record(st)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


for rnd in range(6):
    s0 = state()
    t = burst(5)
    print(f"burst {rnd}: {' '.join('%.3f' % x for x in t)}  before: {s0}  after: {state()}", flush=True)
    t = burst(200)  # ~0.8 s of load
    print(f"  load x200: first {t[0]:.3f} last {t[-1]:.3f} min {min(t):.3f}  {state()}", flush=True)
    time.sleep(3)
