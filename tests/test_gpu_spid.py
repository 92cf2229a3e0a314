"""GPU SPID proper -- coarse-grid skeleton + multilinear lift (SURVEY 8(f)
row 1) -- against the compiled reference's spid() / InterpOperator::apply:
  * the lift M * coarse is bit-identical to InterpOperator::apply;
  * spid() factors (indices, coefficients, coarse skeleton) are bit-identical;
  * the reconstruction M * skel_c * C matches within fp64 reordering;
plus the reference's SPID known-answer tests (proj/tests/test_id_core.cpp:
382-414, proj/tests/python/test_smoke.py:24-30)."""
import numpy as np
import pytest

from conftest import tgv2d

pytestmark = pytest.mark.gpu

SPECS = [([24], [3], None), ([24], [5], [1]), ([20, 20], [2, 2], [1, 1]), ([9, 7], [2, 2], None),
         ([9, 7], [4, 4], None), ([9, 7], [3, 2], [1, 0]), ([16, 16, 16], [3, 2, 3], [1, 0, 1]),
         ([12, 10, 8], [3, 3, 3], None), ([32, 32, 32], [2, 2, 2], None), ([7], [7], [1])]


@pytest.mark.parametrize("dims,strides,per", SPECS)
def test_interp_apply_bitwise(spid, ref, dims, strides, per):
    J = ref.row_indices(dims, strides, per)
    rng = np.random.default_rng(len(J))
    c = np.asfortranarray(rng.standard_normal((len(J), 5)))
    g = spid.interp_apply(dims, strides, c, per)
    assert np.array_equal(g, ref.interp_apply(dims, strides, c, per))


def test_interp_apply_qoi_blocks(spid, ref):
    dims, strides = [16, 16, 16], [2, 2, 2]
    J = ref.row_indices(dims, strides)
    c = np.asfortranarray(np.random.default_rng(1).standard_normal((3 * len(J), 4)))
    g = spid.interp_apply(dims, strides, c, nqoi=3)
    P = 16 ** 3
    for q in range(3):
        assert np.array_equal(g[q * P:(q + 1) * P], ref.interp_apply(dims, strides, c[q * len(J):(q + 1) * len(J)]))


@pytest.mark.parametrize("dims,strides,per", SPECS[:8])
def test_spid_bitwise_vs_reference(spid, ref, orc, dims, strides, per):
    m = int(np.prod(dims))
    a = orc.matmul(orc.seeded_matrix(m, 4, m), orc.seeded_matrix(4, 11, m + 1))
    a = a + 1e-3 * orc.seeded_matrix(m, 11, m + 2)
    nJ = len(ref.row_indices(dims, strides, per))
    for k in sorted({1, min(3, nJ, 11)}):
        g = spid.spid(a, dims, strides, rank=k, periodic=per)
        r = ref.spid(a, dims, strides, rank=k, periodic=per)
        f = g["factors"].base
        assert np.array_equal(f.skeleton_indices, r.indices)
        assert np.array_equal(f.coeffs, r.coeffs)
        assert np.array_equal(f.skeleton, r.skeleton)  # coarse skeleton B(:, I)
        assert f.qr_residual_fro == r.residual_fro
        scale = np.max(np.abs(r.y))
        assert np.max(np.abs(g["approx"] - r.y)) <= 1e-13 * scale


def test_spid_stride1_equals_column_id(spid, orc):
    # test_id_core.cpp:382-392
    a = orc.seeded_matrix(15, 8, 61)
    direct = spid.column_id(a, rank=3)
    single = spid.spid(a, [15], [1], rank=3)
    f = single["factors"].base
    assert np.array_equal(f.skeleton_indices, direct.skeleton_indices)
    assert np.array_equal(f.coeffs, direct.coeffs)
    assert spid.rel_frob_error(spid.reconstruct(direct), single["approx"]) <= 1e-12


def test_spid_exact_on_multilinear_data(spid, orc):
    # test_id_core.cpp:394-414
    st = [99]
    a = np.zeros((63, 5), order="F")
    for c in range(5):
        w0, wx, wy, wxy = (2.0 * (orc.splitmix_next(st) >> 11) * 2.0 ** -53 - 1.0 for _ in range(4))
        for y in range(7):
            for x in range(9):
                a[x + 9 * y, c] = w0 + wx * x + wy * y + wxy * x * y
    for s in (2, 4):
        f = spid.spid(a, [9, 7], [s, s], tol=1e-12)
        assert f["skeleton"].shape[0] == len(spid.row_indices([9, 7], [s, s]))
        assert spid.rel_frob_error(a, f["approx"]) <= 1e-12


def test_spid_tgv_smoke(spid):
    # proj/tests/python/test_smoke.py:24-30
    a = tgv2d((32, 32), steps=40)
    f = spid.spid(a, [32, 32], [2, 2], rank=1, periodic=[True, True])
    assert f["approx"].shape == a.shape
    assert spid.rel_frob_error(a, f["approx"]) <= 5e-2
    stored = f["factors"].stored_entries()
    assert stored == 1 * (16 * 16 + 40)  # k (m_c + n)


def test_spid_errors(spid, orc):
    a = orc.seeded_matrix(24, 5, 1)
    with pytest.raises(spid.SpidError) as e:
        spid.spid(a, [25], [2], rank=1)
    assert e.value.name == "GeometryMismatch"
    with pytest.raises(spid.SpidError) as e:
        spid.spid(a, [24], [0], rank=1)
    assert e.value.name == "BadSubsampleSpec"
    with pytest.raises(spid.SpidError) as e:
        spid.spid(a, [24], [5], rank=1, include_boundary=False)
    assert e.value.name == "ExtrapolationRequired"


def test_lift_and_reconstruct_check_factor_shapes(spid, orc):
    """interp_apply / spid_reconstruct take the coarse row count and the
    coefficient row count through the C ABI and raise DimensionMismatch on
    inconsistent factors (proj/src/interp.cpp:170,179; proj/src/id.cpp:93-94)
    instead of reading past the host buffers; extrapolation is reported
    under its own name (interp.cpp:27-29)."""
    coarse = orc.seeded_matrix(7, 3, 2)  # 24 points, stride 4, boundary: 7 coarse points
    spid.interp_apply([24], [4], coarse)
    with pytest.raises(spid.SpidError) as e:
        spid.interp_apply([24], [4], coarse[:6])
    assert e.value.name == "DimensionMismatch"
    with pytest.raises(spid.SpidError) as e:
        spid.interp_apply([24], [5], orc.seeded_matrix(5, 3, 2), include_boundary=False)
    assert e.value.name == "ExtrapolationRequired"
    a = orc.seeded_matrix(24, 9, 1)
    f = spid.spid(a, [24], [4], rank=2)
    spid.spid_reconstruct(f["factors"])
    base = f["factors"].base
    good_c = base.coeffs
    base.coeffs = good_c[:1]
    with pytest.raises(spid.SpidError) as e:
        spid.spid_reconstruct(f["factors"])
    assert e.value.name == "DimensionMismatch"
    base.coeffs, good_s = good_c, base.skeleton
    base.skeleton = good_s[:5]
    with pytest.raises(spid.SpidError) as e:
        spid.spid_reconstruct(f["factors"])
    assert e.value.name == "DimensionMismatch"
    base.skeleton = good_s


def test_batched_gather_reports_out_of_range_indices(engine):
    """The asynchronous gathers record an index outside the matrix
    (select_columns' IndexOutOfRange, proj/src/dense_matrix.cpp:75) for
    spidgpu_stream_status; valid columns are still gathered."""
    import ctypes as C

    import torch

    from paper_2103_01380_b200 import _native as N

    A = torch.randn((2, 10, 64), dtype=torch.float64, device="cuda")
    idx = torch.tensor([[3, 9], [1, 10]], dtype=torch.int64, device="cuda")  # 10 is out of range
    rank = torch.tensor([2, 2], dtype=torch.int64, device="cuda")
    skel = torch.zeros((2, 2, 64), dtype=torch.float64, device="cuda")
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    engine.h.check(N.lib.spidgpu_gather_batched(engine.h.h, p(A), 64, 10, 64, 640, 2, p(idx), 2, p(rank),
                                                p(skel), 64, 128, None))
    with pytest.raises(N.SpidError) as e:
        engine.stream_status()
    assert e.value.name == "IndexOutOfRange"
    engine.stream_status()  # cleared
    assert torch.equal(skel[0, 0], A[0, 3]) and torch.equal(skel[1, 0], A[1, 1])
    rows = torch.tensor([0, 5, 64], dtype=torch.int64, device="cuda")
    B = torch.empty((2, 10, 3), dtype=torch.float64, device="cuda")
    engine.h.check(N.lib.spidgpu_row_gather_batched(engine.h.h, p(A), 64, 10, 64, 640, 2, p(rows), 3, p(B), 3,
                                                    30, None))
    with pytest.raises(N.SpidError) as e:
        engine.stream_status()
    assert e.value.name == "IndexOutOfRange"
    engine.reserve(64, 10, 2, 48, 8)
