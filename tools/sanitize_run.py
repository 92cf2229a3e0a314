"""Small workloads for compute-sanitizer (memcheck / synccheck / racecheck /
initcheck) over every kernel family of the compress path:

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [part ...]

parts: sketch_tc (one CTA per tile; forced CTA pairs; the slice-split pair
at ell = 80), sketch_dmma (explicit Omega), cpqr (register, generic,
shared/global W, tall TMA ring), gather, verify (TMA and slab), pipeline,
archive. Sizes are kept small: the sanitizer serialises and instruments every
access. Exits non-zero on any Python-side mismatch; the tool reports its own
error summary."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2103_01380_b200 import _native as N  # noqa: E402
from paper_2103_01380_b200.engine import Engine  # noqa: E402
from paper_2103_01380_b200.spid import RankRule  # noqa: E402


def sketch_tc(eng):
    torch.manual_seed(0)
    A = torch.randn((3, 256, 8192), dtype=torch.float64, device="cuda")
    y = eng.sketch(A, 48, seed=1)
    for mode in (2, 0):  # forced CTA pairs, no pairs
        eng.h.check(N.lib.spidgpu_set_option(eng.h.h, N.SPIDGPU_OPT_SKETCH_PAIRS, mode))
        assert torch.equal(eng.sketch(A, 48, seed=1), y)
        eng.sketch(A, 32, seed=1)
    eng.h.check(N.lib.spidgpu_set_option(eng.h.h, N.SPIDGPU_OPT_SKETCH_PAIRS, 1))
    eng.sketch(A, 64, seed=1)
    y80 = eng.sketch(A, 80, seed=1)  # slice-split CTA pairs
    assert torch.isfinite(y80).all()
    torch.cuda.synchronize()


def sketch_dmma(eng):
    torch.manual_seed(1)
    A = torch.randn((2, 100, 4096), dtype=torch.float64, device="cuda")
    om = torch.randn((2, 4096, 30), dtype=torch.float64, device="cuda")
    eng.sketch(A, 30, omega=om)
    torch.cuda.synchronize()


def cpqr(eng):
    torch.manual_seed(2)
    Y = torch.randn((4, 256, 48), dtype=torch.float64, device="cuda")
    eng.cpqr(Y, RankRule.fixed(32))
    eng.h.check(N.lib.spidgpu_set_option(eng.h.h, N.SPIDGPU_OPT_GENERIC_CPQR, 1))
    eng.cpqr(Y, RankRule.fixed(32))
    eng.cpqr(torch.randn((2, 200, 300), dtype=torch.float64, device="cuda"), RankRule.fixed(40))  # W in global
    eng.h.check(N.lib.spidgpu_set_option(eng.h.h, N.SPIDGPU_OPT_GENERIC_CPQR, 0))
    eng.cpqr(torch.randn((2, 64, 512), dtype=torch.float64, device="cuda"), RankRule.fixed(16))  # tall: TMA ring
    torch.cuda.synchronize()


def gather_verify(eng):
    torch.manual_seed(3)
    A = torch.randn((2, 256, 8192), dtype=torch.float64, device="cuda")
    r = eng.compress(A, 48, RankRule.fixed(32), seed=5)
    r.check()
    eng.verify(A, r)
    torch.cuda.synchronize()


def pipeline(eng):
    from paper_2103_01380_b200 import pipeline as PL

    rng = np.random.default_rng(4)
    a = np.asfortranarray(rng.standard_normal((32 * 32, 3)) @ rng.standard_normal((3, 24)))
    cfg = PL.StreamConfig(dims=(32, 32), blocks=(2, 2), strides=(2, 2), time_chunk=8, stage1_rank=3,
                          stage2_tol=1e-6)
    with PL.Pipeline(cfg) as p:
        for j in range(24):
            p.push(a[:, j:j + 1])
        p.finish()
        p.events()


def archive(eng):
    from paper_2103_01380_b200 import archive as AR

    rng = np.random.default_rng(5)
    a = np.asfortranarray(rng.standard_normal((16 * 16 * 8, 2)) @ rng.standard_normal((2, 20)))
    data = AR.compress_field(a, (16, 16, 8), (2, 2, 1), (2, 2, 2), rank=2, periodic=(0, 0, 0), qoi="u",
                             provenance="sanitize")
    AR.decompress(data)


PARTS = {"sketch_tc": sketch_tc, "sketch_dmma": sketch_dmma, "cpqr": cpqr, "gather_verify": gather_verify,
         "pipeline": pipeline, "archive": archive}

if __name__ == "__main__":
    eng = Engine(0)
    for name in (sys.argv[1:] or list(PARTS)):
        PARTS[name](eng)
        torch.cuda.synchronize()
        print("ran", name, flush=True)
