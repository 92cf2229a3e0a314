"""Tall column IDs (rows >= 256, W too large for shared memory, n <= 256): the
CPQR kernel streams W through a TMA ring of row chunks (cpqr.cu, mode 2;
compile-time row lengths 16/32/64/128/256 and the runtime one are all hit).
Same bar as every CPQR path: bit-exact pivots, R, Q, coefficients and
residual against the oracle, including the error exits (the producer warp
must be released on every one of them, or the launch would hang)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _eq(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


@pytest.mark.parametrize("m,n,k", [(4096, 32, 16), (1000, 256, 32), (3001, 7, 5), (2500, 130, 40),
                                   (257, 255, 60), (70000, 3, 3), (5000, 16, 16), (2000, 128, 20),
                                   (1777, 63, 30)])
def test_tall_fixed_rank_bitwise(spid, orc, m, n, k):
    a = orc.seeded_matrix(m, n, 5 + m + n)
    g = spid.column_id(a, rank=k)
    o = orc.column_id(a, rank=k)
    assert g.achieved_rank == o.rank == k
    assert _eq(g.skeleton_indices, o.indices)
    assert _eq(g.coeffs, o.coeffs)
    assert g.qr_residual_fro == o.residual_fro


@pytest.mark.parametrize("m,n", [(4096, 32), (600, 200)])
def test_tall_qr_factors_bitwise(spid, orc, m, n):
    a = orc.seeded_matrix(m, n, 91 + n)
    q = spid.qr(a, rank=12)
    qo = orc.qr(a, rank=12)
    assert _eq(q["q"], qo.q) and _eq(q["r"], qo.r) and _eq(q["pivots"], qo.pivots)


@pytest.mark.parametrize("tol", [1e-2, 1e-6, 1e-12])
def test_tall_tolerance_and_blocked_rules(spid, orc, tol):
    from paper_2103_01380_b200.spid import RankRule

    m, n, r = 2048, 96, 9
    a = orc.matmul(orc.seeded_matrix(m, r, 3), orc.seeded_matrix(r, n, 4))
    a = a + 1e-7 * orc.seeded_matrix(m, n, 5)
    g = spid.column_id(a, tol=tol)
    o = orc.column_id(a, tol=tol)
    assert g.achieved_rank == o.rank
    assert _eq(g.skeleton_indices, o.indices) and _eq(g.coeffs, o.coeffs)
    assert g.qr_residual_fro == o.residual_fro
    gb = spid.column_id(a, rule=RankRule.blocked(40, 4, max(tol, 1e-9)))
    ob = orc.column_id(a, rank=40, tol=max(tol, 1e-9), kstep=4)
    assert gb.achieved_rank == ob.rank
    assert _eq(gb.skeleton_indices, ob.indices) and _eq(gb.coeffs, ob.coeffs)


def test_tall_rank_deficient_and_at_most(spid, orc):
    m, n = 3000, 64
    a = orc.matmul(orc.seeded_matrix(m, 6, 21), orc.seeded_matrix(6, n, 22))
    a[:, 10] = 0.0
    a[:, 40] = a[:, 3]  # exact duplicate: pivot tie order
    g = spid.column_id_at_most(a, 20)
    o = orc.column_id(a, rank=20, at_most=True)
    assert g.achieved_rank == o.rank
    assert _eq(g.skeleton_indices, o.indices) and _eq(g.coeffs, o.coeffs)


def test_tall_error_exits_release_the_producer(spid):
    """Every early exit of the consumers (non-finite input, zero matrix, rank
    unreachable) returns the reference's error instead of hanging."""
    from paper_2103_01380_b200 import SpidError

    def name(fn):
        try:
            fn()
        except SpidError as e:
            return e.name
        return ""

    m, n = 2048, 40
    a = np.random.default_rng(0).standard_normal((m, n))
    bad = a.copy()
    bad[1000, 7] = np.nan
    assert name(lambda: spid.column_id(bad, rank=4)) == "NonFiniteInput"
    assert name(lambda: spid.column_id(np.zeros((m, n)), rank=4)) == "ZeroMatrix"
    low = np.outer(a[:, 0], np.ones(n))
    assert name(lambda: spid.column_id(low, rank=5)) == "RankUnreachable"
    # the handle still works afterwards
    g = spid.column_id(a, rank=4)
    assert g.achieved_rank == 4


def test_tall_batched_statuses_and_parity(engine, orc):
    """Batched device CPQR of 5 tall subdomains, one of them poisoned: the
    others match the oracle bit for bit, the poisoned one reports its error."""
    from paper_2103_01380_b200.spid import RankRule

    rows, n, k = 1500, 120, 24
    mats = [orc.seeded_matrix(rows, n, 300 + s) for s in range(5)]
    mats[2] = mats[2].copy()
    mats[2][17, 5] = np.inf
    Y = torch.stack([torch.from_numpy(np.ascontiguousarray(x.T)) for x in mats]).cuda()
    res = engine.cpqr(Y, RankRule.fixed(k))
    st = res.status.cpu().tolist()
    assert st[2] == 1 and all(st[s] == 0 for s in (0, 1, 3, 4))
    for s in (0, 1, 3, 4):
        o = orc.column_id(mats[s], rank=k)
        assert np.array_equal(res.indices[s].cpu().numpy(), o.indices)
        assert np.array_equal(np.asfortranarray(res.coeffs[s].cpu().numpy().T), o.coeffs)
        assert float(res.residual_fro[s]) == o.residual_fro


@pytest.fixture(params=[1, 0], ids=["pairs", "single"])
def tall_pairs(request, spid):
    """Wide tall inputs (64 < n <= 256, fixed / tolerance rules) run on a
    cluster of two CTAs by default (cpqr_pair.cu); 0 forces one CTA."""
    from paper_2103_01380_b200 import _native as N

    h = spid._h(0)
    h.check(N.lib.spidgpu_set_option(h.h, N.SPIDGPU_OPT_TALL_PAIRS, request.param))
    yield request.param
    h.check(N.lib.spidgpu_set_option(h.h, N.SPIDGPU_OPT_TALL_PAIRS, 1))


@pytest.mark.parametrize("m,n,k", [(4096, 256, 32), (1000, 200, 24), (2500, 130, 40), (3000, 100, 20),
                                   (257, 255, 60), (600, 65, 65)])
def test_tall_pairs_bitwise(tall_pairs, spid, orc, m, n, k):
    """The pair kernel and the single-CTA kernel both equal the oracle bit for
    bit: pivots, coefficients, residual, and Q / R."""
    a = orc.seeded_matrix(m, n, 17 + m + n)
    g = spid.column_id(a, rank=k)
    o = orc.column_id(a, rank=k)
    assert g.achieved_rank == o.rank == k
    assert _eq(g.skeleton_indices, o.indices) and _eq(g.coeffs, o.coeffs)
    assert g.qr_residual_fro == o.residual_fro
    q = spid.qr(a, rank=min(k, 12))
    qo = orc.qr(a, rank=min(k, 12))
    assert _eq(q["q"], qo.q) and _eq(q["r"], qo.r) and _eq(q["pivots"], qo.pivots)


@pytest.mark.parametrize("tol", [1e-1, 1e-6])
def test_tall_pairs_tolerance_and_errors(tall_pairs, spid, orc, tol):
    """Tolerance rule and the error exits through the pair (the peer must
    never be left waiting): rank-deficient input with a strict fixed rank,
    and a non-finite entry in the second CTA's half."""
    from paper_2103_01380_b200 import SpidError

    a = orc.seeded_matrix(3000, 180, 7)
    g = spid.column_id(a, tol=tol)
    o = orc.column_id(a, tol=tol)
    assert g.achieved_rank == o.rank and _eq(g.skeleton_indices, o.indices) and _eq(g.coeffs, o.coeffs)
    low = np.asfortranarray(orc.seeded_matrix(3000, 5, 8) @ orc.seeded_matrix(5, 180, 9))
    with pytest.raises(SpidError) as e:
        spid.column_id(low, rank=40)
    assert e.value.name == "RankUnreachable"
    bad = a.copy()
    bad[1234, 170] = np.nan
    with pytest.raises(SpidError) as e:
        spid.column_id(bad, rank=10)
    assert e.value.name == "NonFiniteInput"
    # the handle still works afterwards
    assert spid.column_id(a, rank=10).achieved_rank == 10
