"""GPU column ID / CPQR (spidgpu_column_id, spidgpu_qr, spidgpu_sub_id)
against the CPU oracle and the compiled reference, plus the reference's own
known-answer tests (proj/tests/test_matrix_core.cpp, test_id_core.cpp,
acceptance.cpp criteria 1 and 6) replayed through the C ABI.

Given the same input matrix the GPU kernel performs the reference's exact
operation sequence, so the bar here is BIT-EXACT equality of pivots, R, Q,
coefficients and residual."""
import numpy as np
import pytest

from conftest import tgv2d

pytestmark = pytest.mark.gpu


def _eq(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


SHAPES = [(3, 3), (7, 2), (9, 6), (14, 9), (15, 10), (16, 11), (20, 12), (33, 17), (48, 256),
          (30, 512), (80, 256), (20, 100), (5, 40), (64, 3), (400, 100)]


@pytest.mark.parametrize("m,n", SHAPES)
def test_column_id_bitwise_vs_oracle(spid, orc, m, n):
    a = orc.seeded_matrix(m, n, 1000 + 7 * m + n)
    for k in sorted({1, min(3, m, n), min(m, n) // 2 or 1, min(m, n)}):
        g = spid.column_id(a, rank=k)
        o = orc.column_id(a, rank=k)
        assert g.achieved_rank == o.rank == k
        assert _eq(g.skeleton_indices, o.indices), (m, n, k)
        assert _eq(g.coeffs, o.coeffs), (m, n, k)
        assert g.qr_residual_fro == o.residual_fro
        assert _eq(g.skeleton, o.skeleton)


@pytest.mark.parametrize("tol", [0.5, 1e-2, 1e-6, 1e-12])
def test_tolerance_rule_bitwise(spid, orc, tol):
    for seed, (m, n) in enumerate([(12, 9), (30, 50), (48, 256)]):
        a = orc.matmul(orc.seeded_matrix(m, 4, seed), orc.seeded_matrix(4, n, seed + 50))
        a = a + 1e-7 * orc.seeded_matrix(m, n, seed + 99)
        g = spid.column_id(a, tol=tol)
        o = orc.column_id(a, tol=tol)
        assert g.achieved_rank == o.rank
        assert _eq(g.skeleton_indices, o.indices) and _eq(g.coeffs, o.coeffs)
        assert g.qr_residual_fro == o.residual_fro


def test_blocked_rule_bitwise(spid, orc):
    from paper_2103_01380_b200.spid import RankRule

    for seed, (m, n, r) in enumerate([(80, 256, 12), (80, 256, 40), (40, 100, 70)]):
        a = orc.matmul(orc.seeded_matrix(m, r, seed), orc.seeded_matrix(r, n, seed + 5))
        a = a + 1e-9 * orc.seeded_matrix(m, n, seed + 9)
        for tol in (1e-3, 1e-6):
            g = spid.column_id(a, rule=RankRule.blocked(64, 8, tol))
            o = orc.column_id(a, rank=64, tol=tol, kstep=8)
            assert g.achieved_rank == o.rank
            assert _eq(g.skeleton_indices, o.indices) and _eq(g.coeffs, o.coeffs)


def test_at_most_bitwise(spid, orc, ref):
    # column_id_at_most: quiet stop at the numerical rank (qr.cpp:22-25)
    a = orc.matmul(orc.seeded_matrix(20, 2, 1), orc.seeded_matrix(2, 15, 2))
    g = spid.column_id_at_most(a, 6)
    o = orc.column_id(a, rank=6, at_most=True)
    r = ref.column_id(a, rank=6, at_most=True)
    assert g.achieved_rank == o.rank == r.rank
    assert _eq(g.coeffs, r.coeffs) and _eq(g.skeleton_indices, r.indices)


@pytest.mark.parametrize("seed", [11, 12, 13, 14])
def test_qr_bitwise_vs_reference(spid, ref, orc, seed):
    a = orc.seeded_matrix(14, 9, seed)
    for k in (1, 4, 9):
        g = spid.qr(a, rank=k)
        r = ref.qr(a, rank=k)
        assert _eq(g["pivots"], r.pivots)
        assert _eq(g["q"], r.q) and _eq(g["r"], r.r)
        assert g["residual_fro"] == r.residual_fro


def test_reference_column_id_bitwise(spid, ref, orc):
    rng = np.random.default_rng(5)
    for rep in range(30):
        m, n = int(rng.integers(2, 60)), int(rng.integers(2, 60))
        a = orc.seeded_matrix(m, n, 5000 + rep)
        k = int(rng.integers(1, min(m, n) + 1))
        g = spid.column_id(a, rank=k)
        r = ref.column_id(a, rank=k)
        assert _eq(g.skeleton_indices, r.indices) and _eq(g.coeffs, r.coeffs)
        assert g.qr_residual_fro == r.residual_fro


def test_sub_id_bitwise_vs_reference(spid, ref, orc):
    cases = [([18], [1], None), ([24], [3], None), ([20, 20], [2, 2], [True, True]),
             ([9, 7], [2, 2], None), ([16, 16, 16], [2, 3, 2], [True, True, True]),
             ([12, 10, 8], [3, 3, 3], None)]
    for ci, (dims, strides, per) in enumerate(cases):
        m = int(np.prod(dims))
        a = orc.seeded_matrix(m, 13, 300 + ci)
        J = ref.row_indices(dims, strides, per)
        assert _eq(spid.row_indices(dims, strides, per), J)
        for k in (1, 3, 6):
            g = spid.sub_id(a, dims, strides, rank=k, periodic=per)
            r = ref.sub_id(a, dims, strides, rank=k, periodic=per)
            assert _eq(g.skeleton_indices, r.indices) and _eq(g.coeffs, r.coeffs)
            assert _eq(g.skeleton, r.skeleton) and g.qr_residual_fro == r.residual_fro


# ---- the reference's known-answer tests, through the GPU -------------------------

def test_kat_identity(spid):
    # test_matrix_core.cpp:11-19
    q = spid.qr(np.eye(2), rank=2)
    assert q["rank"] == 2 and list(q["pivots"]) == [0, 1]
    assert q["r"][0, 0] == 1.0 and q["r"][1, 1] == 1.0 and q["r"][0, 1] == 0.0
    assert q["residual_fro"] == 0.0


def test_kat_pivot_tie_break(spid):
    # test_matrix_core.cpp:21-47
    a = np.zeros((4, 3), order="F")
    a[0, 0] = a[1, 1] = a[0, 2] = a[1, 2] = 1.0
    q = spid.qr(a, rank=2)
    assert q["pivots"][0] == 2 and q["pivots"][1] == 0
    assert q["residual_fro"] <= 1e-14
    rec = q["q"] @ q["r"]
    np.testing.assert_allclose(rec, a[:, q["pivots"]], rtol=1e-12, atol=1e-14)


def test_kat_tolerance_rank_one(spid, orc):
    # test_matrix_core.cpp:49-54
    a = np.outer(orc.seeded_vector(12, 31), orc.seeded_vector(9, 32))
    q = spid.qr(a, tol=1e-10)
    assert q["rank"] == 1
    assert q["residual_fro"] <= 1e-10 * np.linalg.norm(a)


def test_kat_error_names(spid, orc):
    # test_matrix_core.cpp:56-73, test_id_core.cpp:462-466
    from paper_2103_01380_b200 import SpidError

    def name(fn):
        try:
            fn()
        except SpidError as e:
            return e.name
        return ""

    assert name(lambda: spid.qr(np.zeros((3, 3)), rank=1)) == "ZeroMatrix"
    r1 = np.outer(orc.seeded_vector(6, 1), orc.seeded_vector(5, 2))
    assert name(lambda: spid.qr(r1, rank=3)) == "RankUnreachable"
    assert name(lambda: spid.qr(r1, rank=9)) == "RankUnreachable"
    nan = np.zeros((2, 2))
    nan[1, 1] = np.nan
    assert name(lambda: spid.qr(nan, rank=1)) == "NonFiniteInput"
    assert name(lambda: spid.RankRule.tolerance(1.5)) == "BadRankRule"
    a = orc.seeded_matrix(5, 4, 111)
    a[3, 2] = np.inf
    assert name(lambda: spid.column_id(a, rank=2)) == "NonFiniteInput"
    assert name(lambda: spid.column_id(np.zeros((4, 4)), rank=1)) == "ZeroMatrix"


def test_kat_duplicate_columns(spid, orc):
    # test_id_core.cpp:22-33
    u = orc.seeded_vector(7, 3)
    a = np.asfortranarray(np.stack([u, u], axis=1))
    f = spid.column_id(a, rank=1)
    assert list(f.skeleton_indices) == [0]
    assert f.coeffs[0, 0] == 1.0
    assert abs(f.coeffs[0, 1] - 1.0) <= 1e-12
    assert spid.rel_frob_error(a, spid.reconstruct(f)) <= 1e-12


def test_kat_full_rank_and_exact_rank(spid, orc):
    # test_id_core.cpp:35-57
    for seed in (5, 6, 7):
        a = orc.seeded_matrix(9, 6, seed)
        f = spid.column_id(a, rank=6)
        assert f.achieved_rank == 6
        assert spid.rel_frob_error(a, spid.reconstruct(f)) <= 1e-10
    a = orc.matmul(orc.seeded_matrix(8, 3, 42), orc.seeded_matrix(3, 6, 43))
    f = spid.column_id(a, tol=1e-10)
    assert f.achieved_rank == 3
    assert spid.rel_frob_error(a, spid.reconstruct(f)) <= 1e-9


def test_kat_identity_submatrix_exact(spid, orc):
    # test_id_core.cpp:59-68
    a = orc.seeded_matrix(12, 10, 8)
    for k in (1, 4, 7):
        f = spid.column_id(a, rank=k)
        sub = f.coeffs[:, f.skeleton_indices]
        assert _eq(sub, np.eye(k))


def test_acceptance_criterion6_residual_identity(spid, orc):
    # acceptance.cpp:325-344: ||A - A(:,I)C||_F equals the trailing QR residual
    state = [777]
    for rep in range(50):
        m = 8 + orc.splitmix_next(state) % 20
        n = 6 + orc.splitmix_next(state) % 16
        a = orc.seeded_matrix(m, n, 10_000 + rep)
        na = np.linalg.norm(a)
        for k in (1, 3, min(m, n)):
            f = spid.column_id(a, rank=k)
            err = np.linalg.norm(a - spid.reconstruct(f))
            res = f.qr_residual_fro
            if max(err, res) <= 1e-13 * na:
                continue
            assert abs(err - res) / res <= 1e-10


def test_acceptance_criterion1_tgv_cf80(spid):
    # acceptance.cpp:77-114 / test_id_core.cpp:121-130: rank 1, CF exactly 80, err <= 1e-12
    for qoi in ("u1", "u2", "p"):
        a = tgv2d(qoi=qoi)
        f = spid.column_id(a, rank=1)
        assert f.achieved_rank == 1
        stored = f.skeleton.size + f.coeffs.size
        assert stored == 500
        assert spid.compression_factor(400, 100, stored) == 80.0
        assert spid.rel_frob_error(a, spid.reconstruct(f)) <= 1e-12
    # sub_id route with a strided sketch (test_id_core.cpp:121-130)
    a = tgv2d()
    f = spid.sub_id(a, [20, 20], [2, 2], rank=1, periodic=[True, True])
    assert spid.rel_frob_error(a, spid.reconstruct(f)) <= 1e-12


def test_metrics_arithmetic(spid, orc):
    # test_archive_metrics.cpp:39-59
    assert spid.compression_factor(400, 100, 500) == 80.0
    assert abs(spid.compression_factor(262144, 100, 262144 + 100) - 99.9619) < 1e-4 * 99.9619
    assert abs(spid.compression_factor(262144, 100, 10648 + 100) - 2439.0) < 1e-3 * 2439
    a = orc.seeded_matrix(6, 5, 3)
    assert spid.rel_frob_error(a, a) == 0.0
    assert abs(spid.rel_frob_error(a, np.zeros((6, 5))) - 1.0) < 1e-15
    assert abs(spid.rel_frob_error([[3.0, 4.0]], [[0.0, 4.0]]) - 0.6) < 1e-15
    from paper_2103_01380_b200 import SpidError

    with pytest.raises(SpidError) as e:
        spid.compression_factor(4, 4, 0)
    assert e.value.name == "ZeroDenominator"
    with pytest.raises(SpidError) as e:
        spid.rel_frob_error(np.zeros((2, 2)), np.zeros((2, 2)))
    assert e.value.name == "ZeroReference"
    with pytest.raises(SpidError) as e:
        spid.rel_frob_error(a, np.zeros((5, 5)))
    assert e.value.name == "DimensionMismatch"


def test_determinism_bitwise(spid, orc):
    # test_matrix_core.cpp:145-153
    a = orc.seeded_matrix(20, 12, 77)
    q1, q2 = spid.qr(a, rank=6), spid.qr(a, rank=6)
    assert _eq(q1["pivots"], q2["pivots"]) and _eq(q1["q"], q2["q"]) and _eq(q1["r"], q2["r"])


@pytest.mark.parametrize("m,n,k", [(48, 256, 32), (30, 512, 20), (80, 256, 64), (20, 100, 10),
                                   (7, 300, 5), (33, 17, 17)])
def test_both_cpqr_kernels_bitwise(spid, orc, m, n, k):
    """Register-resident and shared/global-W CPQR kernels both reproduce the
    reference bit for bit (SPIDGPU_OPT_GENERIC_CPQR switches between them)."""
    from paper_2103_01380_b200 import _native as N

    h = N.handle(0)
    a = orc.seeded_matrix(m, n, 77 + m + n)
    o = orc.column_id(a, rank=k)
    ot = orc.column_id(a, tol=1e-3)
    try:
        for generic in (0, 1):
            h.check(N.lib.spidgpu_set_option(h.h, N.SPIDGPU_OPT_GENERIC_CPQR, generic))
            g = spid.column_id(a, rank=k)
            assert _eq(g.skeleton_indices, o.indices) and _eq(g.coeffs, o.coeffs), generic
            assert g.qr_residual_fro == o.residual_fro
            gt = spid.column_id(a, tol=1e-3)
            assert _eq(gt.coeffs, ot.coeffs) and gt.achieved_rank == ot.rank
            q = spid.qr(a, rank=k)
            qo = orc.qr(a, rank=k)
            assert _eq(q["q"], qo.q) and _eq(q["r"], qo.r) and _eq(q["pivots"], qo.pivots)
    finally:
        N.lib.spidgpu_set_option(h.h, N.SPIDGPU_OPT_GENERIC_CPQR, 0)


@pytest.mark.parametrize("m,k,n", [(37, 5, 11), (300, 32, 70), (1000, 80, 40)])
def test_reconstruct_bitwise_vs_reference_matmul(spid, orc, ref, m, k, n):
    """reconstruct = the reference's matmul (proj/src/dense_matrix.cpp:38-53)
    bit for bit: separately rounded products and sums in ascending k, zero
    coefficients skipped (an identity block and sparse C included)."""
    s = orc.seeded_matrix(m, k, 3 + m)
    c = orc.seeded_matrix(k, n, 4 + n)
    c[:, : min(k, n)] = np.eye(k)[:, : min(k, n)]
    c[:, -1] = 0.0
    c[k // 2] = 0.0
    got = spid.reconstruct(s, np.asfortranarray(c))
    assert np.array_equal(got, orc.matmul(s, np.asfortranarray(c)))
    assert np.array_equal(got, ref.matmul(s, np.asfortranarray(c)))
