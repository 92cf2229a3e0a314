"""Sketch-sized column IDs (33-48 rows, 128 < n <= 256, fixed / tolerance
rules, one wave of pairs) over a cluster of two CTAs (cpqr_reg_pair.cu; other
shapes keep cpqr_reg.cu with the option on too): each CTA keeps half of
the columns in registers, the pair trades argmax candidates and the pivot
column through distributed shared memory. Same bar as every CPQR path:
bit-exact pivots, R, Q, coefficients and residual against the oracle, with
the pair on and off (the single-CTA cpqr_reg.cu), and every error exit
decided identically in both CTAs (a one-sided exit would hang the peer)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _eq(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


@pytest.fixture(params=[1, 0], ids=["pairs", "single"])
def reg_pairs(request, spid):
    from paper_2103_01380_b200 import _native as N

    h = spid._h(0)
    h.check(N.lib.spidgpu_set_option(h.h, N.SPIDGPU_OPT_REG_PAIRS, request.param))
    yield request.param
    h.check(N.lib.spidgpu_set_option(h.h, N.SPIDGPU_OPT_REG_PAIRS, 1))


@pytest.mark.parametrize("m,n,k", [(48, 256, 32), (48, 200, 32), (40, 129, 20), (36, 256, 16), (33, 180, 33),
                                   (48, 255, 10), (48, 140, 48), (33, 150, 1),
                                   (80, 256, 40), (16, 256, 16)])  # the last two: single-CTA dispatch
def test_regpair_fixed_rank_bitwise(reg_pairs, spid, orc, m, n, k):
    a = orc.seeded_matrix(m, n, 40 + m + n)
    g = spid.column_id(a, rank=k)
    o = orc.column_id(a, rank=k)
    assert g.achieved_rank == o.rank == k
    assert _eq(g.skeleton_indices, o.indices) and _eq(g.coeffs, o.coeffs)
    assert g.qr_residual_fro == o.residual_fro
    q = spid.qr(a, rank=min(k, 12))
    qo = orc.qr(a, rank=min(k, 12))
    assert _eq(q["q"], qo.q) and _eq(q["r"], qo.r) and _eq(q["pivots"], qo.pivots)


@pytest.mark.parametrize("tol", [1e-1, 1e-6, 1e-14])
def test_regpair_tolerance_and_at_most(reg_pairs, spid, orc, tol):
    a = orc.seeded_matrix(48, 230, 71)
    g = spid.column_id(a, tol=tol)
    o = orc.column_id(a, tol=tol)
    assert g.achieved_rank == o.rank
    assert _eq(g.skeleton_indices, o.indices) and _eq(g.coeffs, o.coeffs)
    assert g.qr_residual_fro == o.residual_fro
    low = orc.matmul(orc.seeded_matrix(48, 6, 72), orc.seeded_matrix(6, 230, 73))
    low[:, 150] = low[:, 3]  # an exact duplicate across the two halves: tie order
    g = spid.column_id_at_most(low, 20)
    o = orc.column_id(low, rank=20, at_most=True)
    assert g.achieved_rank == o.rank
    assert _eq(g.skeleton_indices, o.indices) and _eq(g.coeffs, o.coeffs)


def test_regpair_error_exits(reg_pairs, spid, orc):
    """Non-finite input in the second CTA's half, zero matrix, rank
    unreachable: the reference's error, no hang; the handle still works."""
    from paper_2103_01380_b200 import SpidError

    def name(fn):
        try:
            fn()
        except SpidError as e:
            return e.name
        return ""

    a = orc.seeded_matrix(48, 256, 74)
    bad = a.copy()
    bad[30, 200] = np.nan
    assert name(lambda: spid.column_id(bad, rank=8)) == "NonFiniteInput"
    assert name(lambda: spid.column_id(np.zeros((48, 256)), rank=4)) == "ZeroMatrix"
    low = np.asfortranarray(np.outer(a[:, 0], np.ones(256)))
    assert name(lambda: spid.column_id(low, rank=5)) == "RankUnreachable"
    assert spid.column_id(a, rank=8).achieved_rank == 8


def test_regpair_batched_statuses_and_parity(reg_pairs, engine, orc):
    """A batch of 6 subdomains (config 3's 48 x 256 shape), one poisoned: the
    others match the oracle bit for bit, the poisoned one reports its error,
    and the pair and single kernels agree on everything."""
    from paper_2103_01380_b200 import _native as N
    from paper_2103_01380_b200.spid import RankRule

    engine.h.check(N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_REG_PAIRS, reg_pairs))
    try:
        rows, n, k = 48, 256, 32
        mats = [orc.seeded_matrix(rows, n, 500 + s) for s in range(6)]
        mats[4] = mats[4].copy()
        mats[4][7, 140] = np.inf
        Y = torch.stack([torch.from_numpy(np.ascontiguousarray(x.T)) for x in mats]).cuda()
        res = engine.cpqr(Y, RankRule.fixed(k))
        st = res.status.cpu().tolist()
        assert st[4] == 1 and all(st[s] == 0 for s in (0, 1, 2, 3, 5))
        for s in (0, 1, 2, 3, 5):
            o = orc.column_id(mats[s], rank=k)
            assert np.array_equal(res.indices[s].cpu().numpy(), o.indices)
            assert np.array_equal(np.asfortranarray(res.coeffs[s].cpu().numpy().T), o.coeffs)
            assert float(res.residual_fro[s]) == o.residual_fro
    finally:
        engine.h.check(N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_REG_PAIRS, 1))


def test_regpair_repeats_bitwise_full_batch(engine):
    """64 subdomains of config 3's shape, 6 repeats with the pair, 2 without:
    all bitwise identical (a race in the exchange slots or the q transfer
    would show up as a different pivot or coefficient)."""
    from paper_2103_01380_b200 import _native as N
    from paper_2103_01380_b200.spid import RankRule

    torch.manual_seed(9)
    Y = torch.randn((64, 256, 48), dtype=torch.float64, device="cuda")
    rule = RankRule.fixed(32)
    ref, *ref_qr = engine.cpqr(Y, rule, want_qr=True)
    try:
        for pairs in [1] * 6 + [0] * 2:
            engine.h.check(N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_REG_PAIRS, pairs))
            out, *qr = engine.cpqr(Y, rule, want_qr=True)
            for f in ("indices", "coeffs", "rank", "residual_fro", "status"):
                assert torch.equal(getattr(out, f), getattr(ref, f)), (pairs, f)
            for a, b in zip(qr, ref_qr):
                assert torch.equal(a, b), pairs
    finally:
        engine.h.check(N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_REG_PAIRS, 1))
