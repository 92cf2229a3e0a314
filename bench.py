#!/usr/bin/env python
"""SPID compression benchmark (BASELINE.json metric) -- one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Workload: BASELINE config 3, the weak-scaling
configuration the metric is quoted on at 1/2/4/8 GPUs -- every GPU compresses
64 subdomains of 32^3 points x 5 QoIs x 256 snapshots (163840 x 256 fp64,
21.47 GB per GPU) with k=32, p=16 and in-kernel Philox Omega; rank r takes
global blocks [64r, 64r+64) of the config-5 256^3 field, so at 8 GPUs the run
is config 5. A step = the whole compress path (sketch -> CPQR + coefficient
solve -> skeleton gather) over all local subdomains plus the 32-byte NCCL
report reduction. The exact-error verify pass is timed separately
 and reported as `verify`.

--impl reference times the reference's own CPU implementation (oracle/_ref,
compiled from /root/reference/proj/src) on the host cores on a bounded
sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "raw-field GB/s compressed (SPID end-to-end) at 1/2/4/8 B200; CF and rel. error"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FP64_PEAK_PATH = os.path.join(ROOT, "profiles", "fp64_peak.json")
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "sketch_traffic.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-quality", action="store_true")
    ap.add_argument("--no-archive", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(cfg_name, rank, world):
    from paper_2103_01380_b200.configs import CONFIGS, weak_range

    cfg = CONFIGS[cfg_name]
    if cfg.per_gpu_subdomains:
        field, first, count = weak_range(cfg, rank, world)
    else:  # fixed-size configs: contiguous share of the config's own field
        lo, hi = (rank * cfg.subdomains) // world, ((rank + 1) * cfg.subdomains) // world
        field, first, count = cfg, lo, hi - lo
    return cfg, field, first, count


FAMILY = {0: "analytic incompressible TGV (u, v, w, p)", 1: "compressible TGV (rho, u, v, w, E)",
          2: "compressible TGV + 64 seeded Fourier modes (rho, u, v, w, E)"}


def describe(cfg, field, first, count, world):
    """config.workload: the field family, shapes, rank rule and partition."""
    rule = (f"blocked rank rule (steps of {cfg.kstep} up to {cfg.k}, sketch error <= {cfg.tol})"
            if cfg.adaptive else f"fixed rank k={cfg.k}")
    part = ("global blocks dealt round-robin over ranks (heavy = upper half of the block grid, +256 "
            "high-wavenumber modes)" if cfg.adaptive else
            f"global blocks [{cfg.per_gpu_subdomains}r, {cfg.per_gpu_subdomains}r+{cfg.per_gpu_subdomains}) on rank r"
            if cfg.per_gpu_subdomains else f"contiguous block ranges (rank 0: [{first}, {first + count}))")
    return (f"{cfg.name}: {count} subdomains on rank 0 of {cfg.block}^3 x {cfg.qois} QoIs x {cfg.n} "
            f"snapshots ({cfg.m}x{cfg.n} fp64), {rule}, p={cfg.p} (ell={cfg.ell}), in-kernel Philox Omega "
            f"(discretised Gaussian Q/32); {part} of the {field.grid}^3 {FAMILY[field.kind]} field, "
            f"{world} rank(s)")


def _free_port():
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args):
    """`python bench.py --gpus N` (N > 1) outside torchrun: start the N ranks
    ourselves, exactly as the driver's torchrun launch would (one process per
    GPU, rendezvous on 127.0.0.1); rank 0 prints the line."""
    import subprocess

    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def check_world(args):
    """The rank count must be the GPU count asked for: a mismatch would
    report N GPUs' worth of work measured on another number of ranks."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}: launch with "
                                   f"--nproc-per-node {args.gpus} (or run without torchrun and let "
                                   f"bench.py start the ranks)"}), file=sys.stderr, flush=True)
        return False
    return True


def _allreduce(t, op=None):
    """All-reduce on the job's backend: NCCL in place on the device tensor; the
    gloo functional-check mode (BENCH_BACKEND=gloo) goes through the host."""
    import torch.distributed as dist

    op = dist.ReduceOp.SUM if op is None else op
    if dist.get_backend() == "nccl":
        dist.all_reduce(t, op=op)
    else:
        h = t.cpu()
        dist.all_reduce(h, op=op)
        t.copy_(h)


def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


# ---- clocks sampled during the timed region (NVML) ----------------------------
class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device):
        self.samples, self.reasons = [], set()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                bits = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for b, name in self.REASONS.items():
                    if bits & b and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---- the reference CPU path (oracle/_ref) ---------------------------------------
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def reference_inputs(cfg, field, first, count, threads, a_dev=None):
    """A bounded sample of the workload for the CPU reference: one subdomain
    per host thread and the exact Philox Omega_s our kernel uses,
    materialised for the reference's matmul. Inputs only, untimed.

    The reference arm builds both on the CPU (oracle/workload.c, the same
    field generator and Omega definition -- tests/test_workload_oracle.py),
    so its process never loads libspidgpu.so. Our own arm's cpu_baseline
    passes its device-resident A (a_dev) so both sides see the same bits."""
    import oracle

    nsamp = max(1, min(threads, count))
    o = oracle.port()
    if a_dev is None:
        a = o.field_generate(field.field_dict(), first, nsamp, threads=threads)  # (S, n, m)
    else:
        a = a_dev[:nsamp].cpu().numpy()
    om = np.stack([np.ascontiguousarray(o.philox_omega(cfg.seed, first + s, cfg.ell, cfg.m).T)
                   for s in range(nsamp)])  # (S, m, ell) == S column-major ell x m
    return a, om


def reference_time(cfg, a, om, threads):
    """Time the reference CPU compress (oracle/_ref: matmul(Omega_s, A_s) +
    column_id(Y, fixed k) + select_columns(A_s, I), std::thread per subdomain)."""
    import oracle

    if not oracle.ref_available():
        oracle.build()
    secs, ranks = oracle.ref().compress_batch(a, om, cfg.k, threads)
    nsamp = a.shape[0]
    raw = 8.0 * cfg.m * cfg.n * nsamp
    return {"value": raw / secs / 1e9, "unit": "GB/s", "cores": int(threads),
            "kind": "reference", "seconds": secs, "cpu_model": cpu_model(),
            "sample": f"{nsamp} of the workload's subdomains ({cfg.m}x{cfg.n} fp64 each, "
                      f"{raw / 1e9:.2f} GB), one per std::thread, Philox Omega materialised "
                      f"for the reference's matmul; compress = matmul + column_id + "
                      f"select_columns (oracle/_ref built from /root/reference/proj/src, -O3, "
                      f"no -march)",
            "ranks_ok": bool(np.all(ranks == cfg.k))}


def reference_single_core(cfg, a, om):
    """The same compress of ONE subdomain on ONE thread (T = 1)."""
    import oracle

    secs, _ = oracle.ref().compress_batch(a[:1], om[:1], cfg.k, 1)
    return {"value": 8.0 * cfg.m * cfg.n / secs / 1e9, "unit": "GB/s", "cores": 1, "seconds": secs,
            "sample": f"1 subdomain ({cfg.m}x{cfg.n}) on 1 thread"}


def repo_libraries():
    """In-tree shared libraries mapped into this process (evidence of what ran)."""
    libs = set()
    try:
        with open("/proc/self/maps") as f:
            for line in f:
                path = line.split()[-1] if line.strip() else ""
                if path.startswith(ROOT) and ".so" in path:
                    libs.add(os.path.relpath(path, ROOT))
    except OSError:
        pass
    return sorted(libs)


def run_reference(args):
    """--impl reference: rank 0 alone times the reference's own C++ on the
    host cores; other ranks exit. Nothing here loads libspidgpu.so or torch:
    inputs come from the CPU generator in oracle/."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg, field, first, count = workload(args.config, 0, 1)
    threads = os.cpu_count() or 1
    a, om = reference_inputs(cfg, field, first, count, threads)
    vals, cpu = [], None
    for i in range(args.warmup + args.steps):
        cpu = reference_time(cfg, a, om, threads)
        if i >= args.warmup:
            vals.append(cpu["value"])
    value = float(statistics.median(vals)) if vals else cpu["value"]
    cpu["value"] = value
    cpu["t1"] = reference_single_core(cfg, a, om)
    nsamp = a.shape[0]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 8.0 * cfg.m * cfg.n * nsamp / value / 1e6,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{cfg.name}: bounded sample of {nsamp} subdomains of "
                              f"{cfg.m}x{cfg.n} (k={cfg.k}, p={cfg.p}) on {threads} host threads",
                   "subdomains": nsamp, "snapshots": cfg.n, "partition": "one subdomain per host thread",
                   "inputs": "generated on the CPU (oracle/workload.c): same field and Omega definitions"},
        "cpu_baseline": cpu,
        "reference_class": "cpu",
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "libraries_loaded": repo_libraries(),
    }
    print(json.dumps(line), flush=True)
    return 0


# ---- our arm --------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2103_01380_b200 import distributed as D
    from paper_2103_01380_b200.engine import Engine, rule_for

    rank, world, local = dist_env()
    # one process per GPU; local % count only matters for the 1-GPU functional
    # check of the multi-rank path (BENCH_BACKEND=gloo), never for numbers
    backend = os.environ.get("BENCH_BACKEND", "nccl")
    if world > 1 and backend == "nccl" and torch.cuda.device_count() < int(os.environ.get("LOCAL_WORLD_SIZE", world)):
        raise SystemExit(f"{world} NCCL ranks but {torch.cuda.device_count()} visible GPU(s)")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cfg, field, first, count = workload(args.config, rank, world)
    eng = Engine(local)
    dev = eng.dev
    rule = rule_for(cfg)
    if cfg.adaptive:
        # config 4: global subdomains dealt round-robin (distributed.round_robin),
        # heavy = the spatially clustered upper half of the 6x6x6 block grid
        # (block z index >= 3, make_block_domains order), so every GPU gets
        # its share of the expensive blocks; generated one block at a time
        nb = field.grid // field.block
        ids = D.round_robin(field.subdomains, rank, world)
        count = len(ids)
        A = eng.alloc_field(field, count)
        for i, g in enumerate(ids):
            heavy = np.array([1 if g // (nb * nb) >= nb // 2 else 0], dtype=np.uint8)
            eng.generate(field, g, 1, out=A[i:i + 1], heavy=heavy)
        first = 0
    else:
        A = eng.generate(field, first, count)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    res = eng.compress(A, cfg.ell, rule, seed=cfg.seed, subdomain_base=first, want_sketch=True)
    res.check()

    ev_sk = []  # (start, end) events around every sketch launch in the timed region

    def step(timed):
        # the three stages of spidgpu_compress_batched, issued separately so the
        # sketch kernel's own duration can be bracketed with events on its stream
        if timed:
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
        eng.sketch(A, cfg.ell, seed=cfg.seed, subdomain_base=first, out=res.sketch)
        if timed:
            s1.record(stream)
            ev_sk.append((s0, s1))
        eng.h.check(_cpqr_into(eng, res, rule))
        eng.h.check(_gather_into(eng, A, res))
        sums = torch.stack([res.residual_fro.square().sum(), res.rank.sum().double()])
        if world > 1:
            _allreduce(sums)
        return sums

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = eng.launches()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t0.record(stream)
        for _ in range(args.steps):
            step(True)
        t1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = eng.launches() - l0  # spidgpu kernels only (the 2 tiny torch report ops excluded)
    ms = t0.elapsed_time(t1)
    sk_ms = sum(a.elapsed_time(b) for a, b in ev_sk) / len(ev_sk)
    tm = torch.tensor([ms, sk_ms], dtype=torch.float64, device=dev)
    if world > 1:
        _allreduce(tm, op=dist.ReduceOp.MAX)
    ms, sk_ms = float(tm[0]), float(tm[1])
    ms_step = ms / args.steps
    # whole-job bytes: every rank's own count (fixed-size configs need not split evenly)
    cnt = torch.tensor([float(count)], dtype=torch.float64, device=dev)
    if world > 1:
        _allreduce(cnt)
    total_subs = int(cnt[0])
    raw_total = cfg.raw_bytes(total_subs)
    value = raw_total / (ms_step / 1e3) / 1e9

    # verify phase (timed separately, after one untimed call that sizes its
    # workspace) and the report
    eng.verify(A, res)
    torch.cuda.synchronize()
    v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nv = 3
    v0.record(stream)
    for _ in range(nv):
        err2, ref2 = eng.verify(A, res)
    v1.record(stream)
    torch.cuda.synchronize()
    verify_ms = v0.elapsed_time(v1) / nv
    sums = D.local_sums(err2.cpu(), ref2.cpu(), res.rank.cpu(), cfg.m, cfg.n).to(dev)
    report = D.reduce_report(sums)
    vt = torch.tensor([verify_ms], dtype=torch.float64, device=dev)
    if world > 1:
        _allreduce(vt, op=dist.ReduceOp.MAX)
    verify_ms = float(vt[0])

    # roofline of the dominant kernel (the sketch). The Philox-Omega sketch
    # is the exact integer-sliced contraction (sketch_tc.cu): it reads A once
    # and is bound by HBM; the FP64-equivalent flop rate is reported beside
    # it against the DMMA roofline the FP64 kernel was bound by.
    flops = 2.0 * cfg.ell * cfg.m * cfg.n * count
    abytes = 8.0 * cfg.m * cfg.n * count
    fp64 = load_json(FP64_PEAK_PATH) or {}
    peak_tf = fp64.get("dmma_tflops", 37.1)
    achieved_tf = flops / (sk_ms / 1e3) / 1e12
    peaks = load_json(PEAKS_PATH) or {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    achieved_gbs = abytes / (sk_ms / 1e3) / 1e9
    traffic = (load_json(TRAFFIC_PATH) or {}).get(cfg.name + "_i8")
    roofline = {
        "bound": "hbm", "achieved": achieved_gbs, "peak": hbm, "unit": "GB/s",
        "frac": achieved_gbs / hbm, "traffic": traffic,
        "kernel": "sketch_tc_kernel (exact 7-slice integer contraction on tcgen05.mma kind::i8, TMEM accumulators, TMA-staged A)",
        "algorithmic": f"8*m*n = {8.0 * cfg.m * cfg.n:.4g} B of A read once per subdomain x {count} "
                       f"subdomains per launch (Omega generated in-kernel, Y = {8.0 * cfg.ell * cfg.n:.4g} B "
                       f"per subdomain written)",
        "kernel_ms": sk_ms,
        "peak_source": "MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth, burst)",
        "fp64_equivalent": {"tflops": achieved_tf, "dmma_peak_tflops": peak_tf,
                            "frac_of_dmma_roofline": achieved_tf / peak_tf,
                            "peak_source": "profiles/fp64_peak.json (sustained DMMA microbenchmark)"},
    }

    # A/B evidence for the sketch design: the same Philox sketch on the FP64
    # DMMA kernel (identical Omega)
    from paper_2103_01380_b200 import _native as NN

    variants = {}
    for vname, opt in (("dmma_fp64", NN.SPIDGPU_OPT_DMMA_SKETCH),):
        eng.h.check(NN.lib.spidgpu_set_option(eng.h.h, opt, 1))
        try:
            eng.sketch(A, cfg.ell, seed=cfg.seed, subdomain_base=first, out=res.sketch)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(3):
                eng.sketch(A, cfg.ell, seed=cfg.seed, subdomain_base=first, out=res.sketch)
            e1.record(stream)
            torch.cuda.synchronize()
            vms = e0.elapsed_time(e1) / 3
            variants[vname] = {"ms": vms, "a_gbs": abytes / (vms / 1e3) / 1e9}
        finally:
            eng.h.check(NN.lib.spidgpu_set_option(eng.h.h, opt, 0))
    variants["tcgen05_i8 (used)"] = {"ms": sk_ms, "a_gbs": achieved_gbs}
    roofline["sketch_variants"] = variants

    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": describe(cfg, field, first, count, world),
                   "subdomains": int(total_subs), "snapshots": cfg.n,
                   "partition": (f"subdomains dealt round-robin over {world} GPU(s)" if cfg.adaptive else
                                 f"static subdomain ranges over {world} GPU(s)") + ", no data exchange",
                   "l2": "inputs (21.5 GB/GPU) larger than L2 (126 MB); no flush needed"},
        "cf": report.cf, "rel_frob_error": report.rel_frob_error,
        "stored_entries": report.stored_entries,
        "verify": {"ms": verify_ms, "raw_gbs_with_verify":
                   raw_total / ((ms_step + verify_ms) / 1e3) / 1e9},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "roofline": roofline,
    }

    if not args.no_quality:
        line["quality_spid"] = quality_spid(eng, cfg, field, A, first, count, world, stream)
    if not args.no_e2e:
        line["e2e"] = e2e_measure(eng, cfg, A, first, count, rule, args, world)
    if not args.no_archive and world == 1:
        from paper_2103_01380_b200._native import SpidError
        # the archive legs compress the field's u at a fixed rank, strictly,
        # as the reference CLI does: a field whose blocks cannot reach that
        # rank (config 4's quiet blocks) reports the reference's error
        # instead of a number
        for key, leg in (("archive", archive_measure), ("pipeline", pipeline_measure)):
            try:
                line[key] = leg(cfg, A, args)
            except SpidError as e:
                line[key] = {"error": str(e)}
    if world > 1:
        dist.barrier()
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        try:
            threads = os.cpu_count() or 1
            a_h, om_h = reference_inputs(cfg, field, first, count, threads, a_dev=A)
            line["cpu_baseline"] = reference_time(cfg, a_h, om_h, threads)
            line["cpu_baseline"]["t1"] = reference_single_core(cfg, a_h, om_h)
        except Exception as e:  # reported, never fatal
            line["cpu_baseline"] = {"error": repr(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def _cpqr_into(eng, res, rule):
    import ctypes as C

    from paper_2103_01380_b200 import _native as N

    S, n, rows = res.sketch.shape
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    import torch

    return N.lib.spidgpu_cpqr_id_batched(
        eng.h.h, p(res.sketch), rows, n, rows, rows * n, S, C.byref(rule.c()), res.kcap,
        p(res.indices), p(res.coeffs), res.kcap * n, p(res.rank), p(res.residual_fro),
        p(res.status), None, None, None, C.c_void_p(torch.cuda.current_stream().cuda_stream))


def _gather_into(eng, A, res):
    import ctypes as C

    import torch

    from paper_2103_01380_b200 import _native as N

    S, n, m = A.shape
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    return N.lib.spidgpu_gather_batched(eng.h.h, p(A), m, n, m, m * n, S, p(res.indices),
                                        res.kcap, p(res.rank), p(res.skel), m, m * res.kcap,
                                        C.c_void_p(torch.cuda.current_stream().cuda_stream))


def quality_spid(eng, cfg, field, A, first, count, world, stream):
    """The BASELINE quality target ("CF > 100 at rel. error <= 1e-3") on the
    same subdomains: SPID proper -- Gaussian-sketch column
    selection with an adaptive rank (blocked rule, steps of 2 up to 64, sketch
    error <= 3e-4), skeleton stored on the stride-2 coarse grid and lifted
    with the reference's multilinear operator. Untimed quality pass, then a
    timed compress of the same variant (sketch with ell = 80 + CPQR + coarse
    gather)."""
    import torch
    import torch.distributed as dist

    from paper_2103_01380_b200 import distributed as D
    from paper_2103_01380_b200.spid import RankRule

    rule = RankRule.blocked(64, 2, 3e-4)
    ell = 64 + cfg.p
    spec = eng.block_spec(field, 2)
    mc = eng.coarse_rows(spec)
    r = eng.compress(A, ell, rule, seed=cfg.seed, subdomain_base=first, want_skel=False)
    r.check()
    sc = eng.gather_coarse(A, r, spec)
    e2, r2 = eng.verify_coarse(A, r, sc, spec)
    ks = r.rank.double()
    sums = torch.stack([e2.sum(), r2.sum(), (ks * (mc + cfg.n)).sum(),
                        torch.tensor(float(cfg.m) * cfg.n * count, dtype=torch.float64, device=eng.dev)])
    rep = D.reduce_report(sums)
    # timed compress of this variant
    reps = 5
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0.record(stream)
    for _ in range(reps):
        eng.compress(A, ell, rule, seed=cfg.seed, subdomain_base=first, want_skel=False, out=r)
        eng.gather_coarse(A, r, spec)
    t1.record(stream)
    torch.cuda.synchronize()
    ms = torch.tensor([t0.elapsed_time(t1) / reps], dtype=torch.float64, device=eng.dev)
    if world > 1:
        _allreduce(ms, op=dist.ReduceOp.MAX)
    return {"variant": "SPID coarse skeleton (stride 2, trilinear lift) + blocked rank (step 2, "
                       "kmax 64, sketch tol 3e-4), ell = 80",
            "cf": rep.cf, "rel_frob_error": rep.rel_frob_error, "m_c": mc,
            "mean_rank": float(ks.mean()), "max_rank": int(ks.max()),
            "ms_per_step": float(ms[0]),
            "raw_gbs": cfg.raw_bytes(count) * world / (float(ms[0]) / 1e3) / 1e9}


def e2e_measure(eng, cfg, A, first, count, rule, args, world):
    """The same metric through the C-ABI host call (spidgpu_compress_host):
    pinned host A in, host factors out, every copy inside the timed region.

    The pinned sample is sized to the host: at most 40% of the available
    host memory is pinned across all local ranks (8 ranks x 64 subdomains
    would pin ~190 GB); the ranks agree on success before any collective."""
    import psutil
    import torch
    import torch.distributed as dist

    kcap = rule.cap(cfg.ell, cfg.n)
    per_sub = (cfg.m * cfg.n + cfg.m * kcap + cfg.n * kcap) * 8
    avail = psutil.virtual_memory().available
    local_ranks = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    ne = int(min(count, max(1, (0.4 * avail) // (local_ranks * per_sub))))
    ok, err = 1, ""
    try:
        a_host = torch.empty((ne,) + tuple(A.shape[1:]), dtype=torch.float64, pin_memory=True)
        a_host.copy_(A[:ne])
        out = {
            "indices": torch.empty((ne, kcap), dtype=torch.int64, pin_memory=True),
            "coeffs": torch.empty((ne, cfg.n, kcap), dtype=torch.float64, pin_memory=True),
            "skel": torch.empty((ne, kcap, cfg.m), dtype=torch.float64, pin_memory=True),
            "rank": torch.empty(ne, dtype=torch.int64, pin_memory=True),
            "residual_fro": torch.empty(ne, dtype=torch.float64, pin_memory=True),
            "status": torch.empty(ne, dtype=torch.int32, pin_memory=True),
        }
        eng.compress_host(a_host, cfg.ell, rule, seed=cfg.seed, subdomain_base=first, group=2,
                          out=out)  # warm-up (allocates the lane buffers)
        torch.cuda.synchronize()
    except Exception as e:  # host memory / pinning failure: reported, never fatal
        ok, err = 0, repr(e)
    flag = torch.tensor([ok], dtype=torch.int32, device=eng.dev)
    if world > 1:
        _allreduce(flag, op=dist.ReduceOp.MIN)
    if not int(flag[0]):
        return {"error": err or "another rank could not pin its e2e sample"}
    if world > 1:
        dist.barrier()
    t = time.perf_counter()
    for _ in range(args.e2e_steps):
        eng.compress_host(a_host, cfg.ell, rule, seed=cfg.seed, subdomain_base=first, group=2,
                          out=out)
    el = torch.tensor([(time.perf_counter() - t) / args.e2e_steps], dtype=torch.float64,
                      device=eng.dev)
    if world > 1:
        _allreduce(el, op=dist.ReduceOp.MAX)
    sec = float(el[0])
    h2d = a_host.numel() * 8
    d2h = sum(v.numel() * v.element_size() for v in out.values())
    return {"value": cfg.raw_bytes(ne) * world / sec / 1e9, "unit": "GB/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "api": "spidgpu_compress_host (C ABI, pinned host buffers, 2 copy/compute lanes)",
            "subdomains_per_rank": ne, "steps": args.e2e_steps, "ms_per_step": sec * 1e3}


def global_field(A, grid, block, qoi):
    """QoI `qoi` of the block-major batch A [S, n, qois*b^3] as one structured
    field (m = grid^3 rows, axis 0 fastest) in column-major layout, blocks in
    make_block_domains order (proj/src/blocking.cpp:31-98)."""
    import torch

    S, n, _ = A.shape
    b3 = block ** 3
    nb = grid // block
    ar = torch.arange(block, device=A.device)
    i0, i1, i2 = torch.meshgrid(ar, ar, ar, indexing="ij")
    rel = (i0 + grid * i1 + grid * grid * i2).permute(2, 1, 0).reshape(-1)  # local flat, axis 0 fastest
    g = torch.arange(S, device=A.device)
    base = block * (g % nb) + grid * block * ((g // nb) % nb) + grid * grid * block * (g // (nb * nb))
    idx = (base[:, None] + rel[None, :]).reshape(-1)
    G = torch.empty((n, grid ** 3), dtype=torch.float64, device=A.device)
    G[:, idx] = A[:, :, qoi * b3:(qoi + 1) * b3].permute(1, 0, 2).reshape(n, -1)
    return G.T  # m x n, column-major


def archive_measure(cfg, A, args):
    """the reference CLI's `compress --chunk 0` of a whole
    structured field into the SPID archive container (spid_cli.cpp:195-232 +
    archive.cpp encode) and its decompress, on the GPU through the C ABI.
    Reference arm: the same CLI path compiled from the reference sources
    (oracle/_ref), single-threaded as the CLI runs it, on a 64^3 sample whose
    archive must be byte-identical to ours."""
    import ctypes as C

    import torch

    from paper_2103_01380_b200 import _native as N
    from paper_2103_01380_b200 import archive as AR

    grid, block, stride, k = cfg.grid, cfg.block, 2, cfg.k
    field = global_field(A, grid, block, qoi=1)
    m, n = field.shape
    raw = m * n * 8
    h = N.handle(torch.cuda.current_device())
    rr = N.RankRule(N.RULE_FIXED, 0, k, 0, 0.0)
    nb = C.c_int64()
    out = {"workload": f"u of the {cfg.name} field: {grid}^3 x {n} fp64 ({raw / 1e9:.2f} GB), "
                       f"{(grid // block) ** 3} blocks of {block}^3, stride {stride}, rank {k}"}

    def compress(mode, src, on_dev):
        spec = N.archive_spec((grid,) * 3, (grid // block,) * 3, (stride,) * 3, (1, 1, 1), mode,
                              k + cfg.p, cfg.seed, "u", "bench")
        h.check(N.lib.spidgpu_archive_compress(h.h, C.c_void_p(src), m, n, m, 1 if on_dev else 0,
                                               C.byref(spec), C.byref(rr), C.byref(nb)))
        return nb.value

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t) / reps

    host = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
    host.copy_(field.T)
    for name, mode in (("sketch", N.ARCHIVE_SKETCH), ("exact", N.ARCHIVE_EXACT)):
        s_dev = timed(lambda: compress(mode, field.data_ptr(), True), 3)
        s_e2e = timed(lambda: compress(mode, host.data_ptr(), False), 2)
        size = nb.value
        view, ln = C.c_void_p(), C.c_int64()
        h.check(N.lib.spidgpu_archive_view(h.h, C.byref(view), C.byref(ln)))
        data = C.string_at(view.value, ln.value)
        dec = torch.empty((n, m), dtype=torch.float64, device=field.device).T
        s_dec = timed(lambda: AR.decompress(data, out=dec), 3)
        err = float(torch.linalg.norm(dec - field) / torch.linalg.norm(field))
        out[name] = {"archive_bytes": size, "cf": raw / size, "rel_frob_error": err,
                     "device_ms": s_dev * 1e3, "device_gbs": raw / s_dev / 1e9,
                     "e2e": {"value": raw / s_e2e / 1e9, "unit": "GB/s", "ms": s_e2e * 1e3,
                             "h2d_bytes_per_step": raw, "d2h_bytes_per_step": size},
                     "decompress_ms": s_dec * 1e3, "decompress_gbs": raw / s_dec / 1e9}
        if name == "sketch":
            out[name]["ell"] = k + cfg.p
    del host
    # reference CLI path on a 64^3 sub-field (8 blocks), byte parity with ours
    try:
        import oracle
        ref = oracle.ref()
        sg = 2 * block
        sub = field.T.reshape(n, grid, grid, grid)[:, :sg, :sg, :sg]  # [n, z, y, x], x fastest
        a_np = sub.reshape(n, -1).cpu().numpy().T  # m_sub x n, column-major
        t = time.perf_counter()
        rb = ref.compress_field(a_np, (sg,) * 3, (2, 2, 2), (stride,) * 3, rank=k, periodic=(0, 0, 0), qoi="u",
                                provenance="bench")
        t_ref = time.perf_counter() - t
        t = time.perf_counter()
        ref.archive_decompress(rb)
        t_ref_dec = time.perf_counter() - t
        ours = AR.compress_field(a_np, (sg,) * 3, (2, 2, 2), (stride,) * 3, rank=k, periodic=(0, 0, 0),
                                 qoi="u", provenance="bench")
        out["reference"] = {"kind": "reference", "cores": 1,
                            "sample": f"{sg}^3 x {n} sub-field, 8 blocks (spid CLI batch path, oracle/_ref)",
                            "compress_gbs": a_np.nbytes / t_ref / 1e9, "compress_s": t_ref,
                            "decompress_gbs": a_np.nbytes / t_ref_dec / 1e9,
                            "bytes_identical": ours == rb}
    except Exception as e:  # reported, never fatal
        out["reference"] = {"error": repr(e)}
    return out


def pipeline_measure(cfg, A, args):
    """the in-situ streaming two-stage compressor
    (run_pipeline, proj/src/pipeline.cpp:104-294) on the GPU: the u field of
    the workload pushed one snapshot at a time (as a solver would produce
    them), chunks of 32 snapshots, stage-1 rank 16, stage-2 tolerance 1e-5,
    stride-2 coarse skeletons. Reference arm: run_pipeline itself (oracle/_ref)
    with one TaskPool worker per host thread on a 64^3 sample, which must give
    the byte-identical archive."""
    import torch

    from paper_2103_01380_b200 import archive as AR
    from paper_2103_01380_b200 import pipeline as PL

    grid, block = cfg.grid, cfg.block
    T, k1, tol2 = 32, 16, 1e-5
    field = global_field(A, grid, block, qoi=1)  # m x n column-major
    m, n = field.shape
    raw = m * n * 8
    frames = field.T  # [n, m]: frame j contiguous
    pc = PL.StreamConfig(dims=(grid,) * 3, blocks=(grid // block,) * 3, strides=(2, 2, 2), time_chunk=T,
                         stage1_rank=k1, stage2_tol=tol2, periodic=(1, 1, 1), qoi="u", provenance="bench")

    import ctypes as C

    from paper_2103_01380_b200 import _native as N

    def run(src, sync=False):
        """push every frame + spidgpu_stream_finish (the archive lands in the
        handle's pinned buffer) -- timed; the copy into a Python bytes object
        (first-touch page faults of 60 MB, ~27 ms) is not the library's work
        and happens after the clock stops. Device frames are always read
        asynchronously; host frames with sync=False too (they stay resident
        and unmodified until finish, so the copies queue back to back), with
        sync=True every push waits for its frame's copy"""
        with PL.Pipeline(pc) as p:
            t = time.perf_counter()
            for j in range(n):
                p.push(src[j], sync=sync)
            nb = C.c_int64()
            p._check(N.lib.spidgpu_stream_finish(p.s, C.byref(nb)))
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            view, ln = C.c_void_p(), C.c_int64()
            p.h.check(N.lib.spidgpu_archive_view(p.h.h, C.byref(view), C.byref(ln)))
            return C.string_at(view.value, ln.value), p.stats(), dt

    # median of 5 timed runs per source after one warm-up: the host-frame run
    # is a chain of 256 synchronous PCIe copies and swings with the host, and
    # on this pool even device-frame runs see occasional multi-ms host stalls
    run(frames)
    torch.cuda.synchronize()
    runs = sorted((run(frames) for _ in range(5)), key=lambda r: r[2])
    data, st, s_dev = runs[2]
    host = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
    host.copy_(frames)
    hf = host.numpy()
    runs_h = sorted((run(hf) for _ in range(5)), key=lambda r: r[2])
    data_h, _, s_host = runs_h[2]
    # synchronous host pushes (each waits for its own frame's copy), for comparison
    data_hs, _, s_host_sync = sorted((run(hf, True) for _ in range(3)), key=lambda r: r[2])[1]
    del host, runs, runs_h
    dec = torch.empty((n, m), dtype=torch.float64, device=field.device).T
    AR.decompress(data, out=dec)
    err = float(torch.linalg.norm(dec - field) / torch.linalg.norm(field))
    out = {"workload": f"u of the {cfg.name} field, {grid}^3 x {n} snapshots pushed one per call, "
                       f"{(grid // block) ** 3} blocks, stride 2, time_chunk {T}, stage-1 rank {k1}, "
                       f"stage-2 tol {tol2}",
           "archive_bytes": len(data), "cf": raw / len(data), "rel_frob_error": err,
           "device_frames": {"ms": s_dev * 1e3, "gbs": raw / s_dev / 1e9,
                             "snapshots_per_s": n / s_dev},
           "e2e": {"value": raw / s_host / 1e9, "unit": "GB/s", "ms": s_host * 1e3,
                   "h2d_bytes_per_step": raw, "d2h_bytes_per_step": len(data_h),
                   "sync_push": {"value": raw / s_host_sync / 1e9, "ms": s_host_sync * 1e3},
                   "api": "spidgpu_stream_push per snapshot from pinned host memory (asynchronous pushes: the "
                          "frames stay unmodified until finish; sync_push = each push waits for its frame's "
                          "copy) + spidgpu_stream_finish (archive D2H into the handle's pinned buffer; the "
                          "Python bytes copy is untimed)"},
           "stage1_ms": st["stage1_ms"], "stage2_ms": st["stage2_ms"],
           "host_and_device_identical": data == data_h and data == data_hs}
    try:
        import oracle
        ref = oracle.ref()
        sg = 2 * block
        sub = field.T.reshape(n, grid, grid, grid)[:, :sg, :sg, :sg]
        a_np = sub.reshape(n, -1).cpu().numpy().T
        threads = os.cpu_count() or 1
        t = time.perf_counter()
        rb, _ = ref.run_pipeline(a_np, (sg,) * 3, (2, 2, 2), (2, 2, 2), T, k1, tol2, periodic=(0, 0, 0),
                                 workers=threads, qoi="u", provenance="bench")
        t_ref = time.perf_counter() - t
        ours = PL.run_pipeline(a_np, PL.StreamConfig(dims=(sg,) * 3, blocks=(2, 2, 2), strides=(2, 2, 2),
                                                     time_chunk=T, stage1_rank=k1, stage2_tol=tol2,
                                                     periodic=(0, 0, 0), qoi="u", provenance="bench"))
        out["reference"] = {"kind": "reference", "cores": threads,
                            "sample": f"{sg}^3 x {n} sub-field, 8 blocks, run_pipeline with {threads} workers",
                            "gbs": a_np.nbytes / t_ref / 1e9, "seconds": t_ref, "bytes_identical": ours == rb}
    except Exception as e:  # reported, never fatal
        out["reference"] = {"error": repr(e)}
    return out


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch(args)
    if not check_world(args):
        return 2
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
