"""Race and bounds evidence without compute-sanitizer (closed on this GPU
pool: profiles/r02_sanitizer.txt). A data race in the asynchronous
pipelines (TMA rings, mbarrier hand-offs, st.async between cluster CTAs,
TMEM flushes) shows up as run-to-run differences of results that are
otherwise bitwise deterministic; an out-of-bounds store shows up in guard
zones around every output. Both are checked here on full-size grids."""
import pytest
import torch

pytestmark = pytest.mark.gpu

GUARD = 4096  # doubles of NaN-poisoned slack on each side of an output


def _guarded(shape, dtype=torch.float64):
    n = 1
    for d in shape:
        n *= d
    buf = torch.full((n + 2 * GUARD,), float("nan") if dtype.is_floating_point else -7, dtype=dtype, device="cuda")
    return buf, buf[GUARD:GUARD + n].view(shape)


def _guards_intact(buf):
    lo, hi = buf[:GUARD], buf[-GUARD:]
    if buf.dtype.is_floating_point:
        return bool(torch.isnan(lo).all() and torch.isnan(hi).all())
    return bool((lo == -7).all() and (hi == -7).all())


@pytest.fixture(scope="module")
def field(engine):
    from paper_2103_01380_b200.configs import CONFIGS

    A = engine.generate(CONFIGS["cfg5"], 8, 24)  # 24 config-3 subdomains (8 GB)
    torch.cuda.synchronize()
    return A


@pytest.mark.parametrize("ell,pairs", [(48, 1), (48, 2), (64, 1), (80, 1), (30, 0)])
def test_sketch_repeats_bitwise_and_stays_in_bounds(engine, field, ell, pairs):
    """One CTA per tile (48, 30), forced tile pairs (48, 2), default pairs
    (64), the slice-split pair (80): 8 repeats bitwise identical, and no
    store outside Y."""
    from paper_2103_01380_b200 import _native as N

    engine.h.check(N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_SKETCH_PAIRS, pairs))
    try:
        S, n, _ = field.shape
        buf, Y = _guarded((S, n, ell))
        engine.sketch(field, ell, seed=3, out=Y)
        ref = Y.clone()
        for _ in range(8):
            engine.sketch(field, ell, seed=3, out=Y)
            assert torch.equal(Y, ref)
        torch.cuda.synchronize()
        assert _guards_intact(buf) and torch.isfinite(ref).all()
    finally:
        engine.h.check(N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_SKETCH_PAIRS, 1))


def test_compress_verify_repeats_bitwise_and_in_bounds(engine, field):
    """The whole compress step (sketch -> CPQR -> gather) and verify, 5
    repeats: factors and error terms bitwise identical; guard zones of the
    skeleton, coefficient and error outputs intact."""
    from paper_2103_01380_b200.engine import CompressResult
    from paper_2103_01380_b200.spid import RankRule

    S, n, m = field.shape
    kcap = 32
    bs, skel = _guarded((S, kcap, m))
    bc, coeffs = _guarded((S, n, kcap))
    bi, idx = _guarded((S, kcap), torch.int64)
    r = CompressResult(idx, coeffs, torch.zeros(S, dtype=torch.int64, device="cuda"),
                       torch.zeros(S, dtype=torch.float64, device="cuda"),
                       torch.zeros(S, dtype=torch.int32, device="cuda"), skel, None, kcap, m, n)
    outs = []
    for _ in range(5):
        engine.compress(field, 48, RankRule.fixed(32), seed=9, out=r)
        e2, r2 = engine.verify(field, r)
        outs.append((r.indices.clone(), r.coeffs.clone(), r.skel.clone(), e2.clone(), r2.clone()))
    torch.cuda.synchronize()
    r.check()
    for o in outs[1:]:
        assert all(torch.equal(a, b) for a, b in zip(o, outs[0]))
    assert _guards_intact(bs) and _guards_intact(bc) and _guards_intact(bi)


@pytest.mark.parametrize("S,n,rows", [(16, 256, 4096), (64, 130, 2500), (64, 200, 1000)])
def test_tall_cpqr_repeats_bitwise(engine, S, n, rows):
    """The TMA-ring column ID (rows >= 256): W streamed through shared memory
    by a producer warp; by default over CTA pairs (argmax exchange, the pivot
    column loaded and divided in both CTAs). 5 repeats with pairs on, then 2
    with pairs off (the single-CTA kernel), all bitwise identical."""
    from paper_2103_01380_b200 import _native as N
    from paper_2103_01380_b200.spid import RankRule

    torch.manual_seed(4 + n)
    Y = torch.randn((S, n, rows), dtype=torch.float64, device="cuda")
    rule = RankRule.fixed(32)
    ref, *ref_qr = engine.cpqr(Y, rule, want_qr=True)
    runs = [1] * 5 + [0] * 2
    try:
        for pairs in runs:
            engine.h.check(N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_TALL_PAIRS, pairs))
            out, *qr = engine.cpqr(Y, rule, want_qr=True)
            for f in ("indices", "coeffs", "rank", "residual_fro", "status"):
                assert torch.equal(getattr(out, f), getattr(ref, f)), (pairs, f)
            for a, b in zip(qr, ref_qr):  # pivots, R, Q
                assert torch.equal(a, b), pairs
    finally:
        engine.h.check(N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_TALL_PAIRS, 1))
