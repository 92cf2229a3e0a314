"""CPU: pin the oracle restatement (oracle/spid_oracle.c).

1. against the golden fixtures generated from the REFERENCE itself
   (tests/golden/reference_cases.npz, made by tests/golden/make_golden.py
   from oracle/_ref) -- bit-exact;
2. against oracle/_ref directly when it is built (this container) -- bit-exact
   on fresh seeded cases;
3. against the reference's own known-answer tests (proj/tests/*.cpp)."""
import hashlib
import os

import numpy as np
import pytest

from conftest import tgv2d

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_cases.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def sha(a):
    return np.frombuffer(hashlib.sha256(np.asfortranarray(a).tobytes(order="F")).digest(),
                         dtype=np.uint8)


def test_golden_column_id_and_qr(orc, gold):
    keys = sorted({k.rsplit("_", 1)[0] for k in gold.files if k.startswith("cid_") and k.endswith("_seed")})
    assert len(keys) >= 25
    for key in keys:
        seed, m, n, k = (int(x) for x in gold[key + "_seed"])
        a = orc.seeded_matrix(m, n, seed)
        assert np.array_equal(sha(a), gold[key + "_a_sha"]), key  # SplitMix64 inputs pinned
        f = orc.column_id(a, rank=k)
        assert np.array_equal(f.indices, gold[key + "_indices"]), key
        assert np.array_equal(f.coeffs, gold[key + "_coeffs"]), key
        assert f.residual_fro == gold[key + "_resid"][0]
        q = orc.qr(a, rank=k)
        assert np.array_equal(q.pivots, gold[key + "_pivots"])
        assert np.array_equal(q.r, gold[key + "_r"]) and np.array_equal(q.q, gold[key + "_q"])


def test_golden_tolerance(orc, gold):
    for si in range(3):
        key = f"tol_{si}"
        a = orc.matmul(orc.seeded_matrix(25, 4, 60 + si), orc.seeded_matrix(4, 30, 70 + si))
        a = a + 1e-7 * orc.seeded_matrix(25, 30, 80 + si)
        assert np.array_equal(a, gold[key + "_a"])
        f = orc.column_id(a, tol=float(gold[key + "_tol"][0]))
        assert np.array_equal(f.indices, gold[key + "_indices"])
        assert np.array_equal(f.coeffs, gold[key + "_coeffs"])


def test_golden_sub_id_rows(gold):
    from paper_2103_01380_b200.spid import row_indices

    for si in range(4):
        key = f"sub_{si}"
        dims = list(gold[key + "_dims"])
        strides = list(gold[key + "_strides"])
        per = [bool(x) for x in gold[key + "_periodic"]]
        assert np.array_equal(row_indices(dims, strides, per), gold[key + "_rows"])


def test_golden_sub_id_via_port(orc, gold):
    # sub_id = column_id on A(J,:) + fine skeleton (id.cpp:54-60)
    for si in range(4):
        key = f"sub_{si}"
        m = int(np.prod(gold[key + "_dims"]))
        a = orc.seeded_matrix(m, 13, int(gold[key + "_seed"][0]))
        assert np.array_equal(sha(a), gold[key + "_a_sha"])
        b = np.asfortranarray(a[gold[key + "_rows"], :])
        f = orc.column_id(b, rank=3)
        assert np.array_equal(f.indices, gold[key + "_indices"])
        assert np.array_equal(f.coeffs, gold[key + "_coeffs"])


def test_golden_gaussian_sketch(orc, gold):
    for si in range(2):
        key = f"sk_{si}"
        m, n, ell, sa, so = (int(x) for x in gold[key + "_shape"])
        a = orc.seeded_matrix(m, n, sa)
        om = orc.gaussian(ell, m, so)
        assert np.array_equal(sha(a), gold[key + "_a_sha"])
        assert np.array_equal(sha(om), gold[key + "_omega_sha"])
        f = orc.sketch_id(a, om, rank=int(gold[key + "_k"][0]))
        assert np.array_equal(f.y, gold[key + "_y"])  # matmul restatement bit-exact
        assert np.array_equal(f.indices, gold[key + "_indices"])
        assert np.array_equal(f.coeffs, gold[key + "_coeffs"])


def test_port_vs_ref_bitwise_fresh(orc, ref):
    rng = np.random.default_rng(11)
    for rep in range(40):
        m, n = int(rng.integers(2, 50)), int(rng.integers(2, 50))
        a = orc.seeded_matrix(m, n, 70_000 + rep)
        k = int(rng.integers(1, min(m, n) + 1))
        p, r = orc.column_id(a, rank=k), ref.column_id(a, rank=k)
        assert np.array_equal(p.indices, r.indices) and np.array_equal(p.coeffs, r.coeffs)
        assert p.residual_fro == r.residual_fro
        tol = float(10.0 ** rng.uniform(-12, -1))
        p, r = orc.column_id(a, tol=tol), ref.column_id(a, tol=tol)
        assert np.array_equal(p.coeffs, r.coeffs)
        p, r = orc.column_id(a, rank=k, at_most=True), ref.column_id(a, rank=k, at_most=True)
        assert np.array_equal(p.coeffs, r.coeffs)


def test_port_matmul_vs_ref(orc, ref):
    a = orc.gaussian(20, 3000, 5)
    b = orc.seeded_matrix(3000, 40, 6)
    b[7, :] = 0.0  # exercises the zero skip of dense_matrix.cpp:47
    assert np.array_equal(orc.matmul(a, b), ref.matmul(a, b))


# ---- reference KATs on the oracle --------------------------------------------------

def test_kat_identity_and_tie_break(orc):
    q = orc.qr(np.eye(2), rank=2)
    assert list(q.pivots) == [0, 1] and q.r[0, 0] == 1.0 and q.r[0, 1] == 0.0
    assert q.residual_fro == 0.0
    a = np.zeros((4, 3), order="F")
    a[0, 0] = a[1, 1] = a[0, 2] = a[1, 2] = 1.0
    q = orc.qr(a, rank=2)
    assert q.pivots[0] == 2 and q.pivots[1] == 0


def test_kat_error_names(orc):
    import oracle

    def name(fn):
        try:
            fn()
        except oracle.OracleError as e:
            return e.name
        return ""

    assert name(lambda: orc.qr(np.zeros((3, 3)), rank=1)) == "ZeroMatrix"
    r1 = np.outer(orc.seeded_vector(6, 1), orc.seeded_vector(5, 2))
    assert name(lambda: orc.qr(r1, rank=3)) == "RankUnreachable"
    assert name(lambda: orc.qr(r1, rank=9)) == "RankUnreachable"
    nan = np.zeros((2, 2))
    nan[1, 1] = np.nan
    assert name(lambda: orc.qr(nan, rank=1)) == "NonFiniteInput"
    assert name(lambda: orc.qr(r1, tol=1.5)) == "BadRankRule"
    assert name(lambda: orc.solve_upper(np.array([[1.0, 2.0], [0.0, 0.0]]), np.ones((2, 1)))) == \
        "SingularPivot"
    assert name(lambda: orc.compression_factor(4, 4, 0)) == "ZeroDenominator"
    assert name(lambda: orc.rel_frob_error(np.zeros((2, 2)), np.zeros((2, 2)))) == "ZeroReference"


def test_kat_solve_and_metrics(orc):
    x = orc.solve_upper(np.array([[2.0, 1.0], [0.0, 4.0]]), np.array([[3.0], [8.0]]))
    assert np.allclose(x[:, 0], [0.5, 2.0])
    assert orc.compression_factor(400, 100, 500) == 80.0
    assert abs(orc.rel_frob_error(np.array([[3.0, 4.0]]), np.array([[0.0, 4.0]])) - 0.6) < 1e-15


def test_kat_residual_identity_criterion6(orc):
    state = [777]
    for rep in range(50):
        m = 8 + orc.splitmix_next(state) % 20
        n = 6 + orc.splitmix_next(state) % 16
        a = orc.seeded_matrix(m, n, 20_000 + rep)
        for k in (1, 3, min(m, n)):
            f = orc.column_id(a, rank=k)
            e2, _ = orc.error_terms(a, f.skeleton, f.coeffs)
            err, res = np.sqrt(e2), f.residual_fro
            if max(err, res) <= 1e-13 * np.linalg.norm(a):
                continue
            assert abs(err - res) / res <= 1e-10


def test_kat_tgv_cf80(orc):
    for qoi in ("u1", "u2", "p"):
        a = tgv2d(qoi=qoi)
        f = orc.column_id(a, rank=1)
        stored = f.skeleton.size + f.coeffs.size
        assert orc.compression_factor(400, 100, stored) == 80.0
        e2, r2 = orc.error_terms(a, f.skeleton, f.coeffs)
        assert np.sqrt(e2 / r2) <= 1e-12


def test_blocked_rule_prefix_property(orc):
    """Greedy CPQR prefixes equal fixed-k runs."""
    a = orc.matmul(orc.seeded_matrix(80, 30, 1), orc.seeded_matrix(30, 200, 2))
    a = a + 1e-6 * orc.seeded_matrix(80, 200, 3)
    fb = orc.column_id(a, rank=64, tol=1e-3, kstep=8)
    assert fb.rank % 8 == 0 and 8 <= fb.rank <= 64
    ff = orc.column_id(a, rank=fb.rank)
    assert np.array_equal(fb.indices, ff.indices) and np.array_equal(fb.coeffs, ff.coeffs)
    # the stop criterion: residual_fro / ||Y||_F <= tol at rank, not at rank-8
    assert fb.residual_fro <= 1e-3 * np.linalg.norm(a)
    if fb.rank > 8:
        prev = orc.column_id(a, rank=fb.rank - 8)
        assert prev.residual_fro > 1e-3 * np.linalg.norm(a) * (1 - 1e-12)
