"""The exact integer-sliced sketch, which runs every Philox-Omega sketch:
Y = Omega A with Omega = Q/32 integer-valued, A split into 7 byte slices of a
per-column fixed point, each slice contracted exactly in int32 on
tcgen05.mma kind::i8 with TMEM accumulators (csrc/sketch_tc.cu). Every test
runs twice: default CTA mode and forced CTA pairs (clusters of two sharing
each stage's Omega tile).

Accuracy contract (csrc/sketch_tc.cu header). Every entry x
of A is rounded once, to the fixed point of its epoch -- a multiple of
2^(E-50) with 2^E <= 16 * (the largest |A| of its 4096-row segment) -- and
everything after that is exact integer arithmetic until one fp64 conversion
per epoch and a fixed-order fp64 sum of the segment partials. So per entry
    |Y - Y_exact|(i,j) <= 2^-47 sum_k |Omega(i,k)| M_j(k) + (nseg + 2) u (|Omega||A|)(i,j)
with M_j(k) the largest |A(., j)| in row k's segment (4096 rows; 8192 with
two partials per segment for the single-pass ell in (64, 80]), u = 2^-53 (tested on
every case below against the product in extended precision, np.longdouble).
The reference sketch is the sequential fp64 matmul
(proj/src/dense_matrix.cpp:38-53), whose own per-entry bound is
    |fl(Y) - Y|(i,j) <= gamma_m (|Omega||A|)(i,j),  gamma_m = m u / (1 - m u);
for data whose columns are not dominated by a few huge entries (every
normal-distributed case below, m >= 1000) our error is also inside gamma_m,
i.e. no worse than the reference's own rounding can be; it is checked there,
and against the oracle's fp64 matmul within the sum of both bounds. The
adversarial columns (a spike then a long tiny tail inside one segment, a
1e-12 block after O(1) rows, alternating scales, exponent growth) are where
the 51-bit fixed point and fp64 differ; the magnitude fallback restarts an
epoch whose rows drop 2^24 below its scale, so a spike cannot coarsen them.

Batch independence: Y_s is bitwise the same whatever batch it is sketched in,
with any SM cap, pair mode or grouping."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


def _host(t):
    return np.asfortranarray(t.detach().cpu().numpy().T)


def _gamma(m):
    return m * U / (1.0 - m * U)


def _dmma(engine, on):
    from paper_2103_01380_b200 import _native as N

    engine.h.check(N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_DMMA_SKETCH, int(on)))


def _pairs(engine, mode):
    from paper_2103_01380_b200 import _native as N

    engine.h.check(N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_SKETCH_PAIRS, mode))


@pytest.fixture(params=["tc", "tc_pairs"], autouse=True)
def kernel(request, engine):
    """tcgen05 sketch with one CTA per column tile for up to 64 rows (the
    default), or with CTA pairs wherever the column tiles pair up."""
    _pairs(engine, 2 if request.param == "tc_pairs" else 1)
    yield request.param
    _pairs(engine, 1)


def _segments(ell):
    """(rows per segment, partials per segment) of the passes sketching ell
    rows (api.cu do_sketch: one pass up to 80 rows, else even passes of whole
    16-row groups): 4096 and 1, or for passes of 65-80 rows, run by the
    slice-split CTA pair, 8192 and 2 (csrc/sketch_tc.cu)."""
    passes = -(-ell // 80)
    width = ell if passes == 1 else min(80, 16 * -(-(-(-ell // passes)) // 16))
    return (8192, 2) if width > 64 else (4096, 1)


def _contract(om, a):
    """The per-entry bound of the fixed-point sketch (see the module doc)."""
    m = a.shape[0]
    seg_rows, halves = _segments(om.shape[0])
    nseg = -(-m // seg_rows)
    M = np.empty_like(a)
    for g in range(nseg):
        blk = np.abs(a[g * seg_rows:(g + 1) * seg_rows])
        M[g * seg_rows:(g + 1) * seg_rows] = blk.max(axis=0, keepdims=True)
    B = np.abs(om) @ np.abs(a)
    return (2.0 ** -47 * (np.abs(om) @ M) + (halves * nseg + 2) * U * B) * (1 + 1e-9), B


def _bound_check(y, om, a, exact=True, gamma=False):
    """Contract vs the extended-precision product (and, with gamma=True, the
    fp64 dot-product bound gamma_m); against the oracle's fp64 matmul within
    contract + gamma_m. Finite columns only. Returns the worst ratio to the
    contract."""
    import oracle

    m = a.shape[0]
    fin = np.all(np.isfinite(a), axis=0)
    a_f = a[:, fin]
    y_f = y[:, fin]
    cb, B = _contract(om, a_f)
    g = _gamma(m) * B * (1 + 1e-9)
    y_ref = oracle.port().matmul(om, np.asfortranarray(a_f))
    d = np.abs(y_f - y_ref)
    assert np.all(d <= cb + g), float(np.max(d / np.maximum(cb + g, 1e-300)))
    worst = 0.0
    if exact:
        yx = om.astype(np.longdouble) @ a_f.astype(np.longdouble)
        d = np.abs(y_f.astype(np.longdouble) - yx)
        assert np.all(d <= cb), float(np.max(d / np.maximum(cb, 1e-300)))
        worst = float(np.max(d / np.maximum(cb, 1e-300)))
        if gamma:
            assert np.all(d <= g), float(np.max(d / np.maximum(g, 1e-300)))
    return worst


def _check(engine, spid, A, ell, seed, base, exact=True, gamma=False):
    Y = engine.sketch(A, ell, seed=seed, subdomain_base=base)
    torch.cuda.synchronize()
    S, n, m = A.shape
    worst = 0.0
    for s in range(S):
        om = spid.philox_omega(seed, base + s, ell, m)
        worst = max(worst, _bound_check(_host(Y[s]), om, _host(A[s]), exact, gamma))
    return Y, worst


def test_omega_is_the_discretised_gaussian(spid):
    om = spid.philox_omega(5, 3, 48, 20000)
    q = om * 32
    assert np.array_equal(q, np.rint(q)) and np.abs(q).max() <= 117
    assert abs(om.mean()) < 0.01 and abs(om.std() - 1.0) < 0.01
    # 16-bit Philox halves -> all 4096 quantiles reachable: many distinct values
    assert len(np.unique(q)) > 150


@pytest.mark.parametrize("m,n,ell", [(6000, 130, 48), (16384, 100, 20), (1000, 37, 30),
                                     (2048, 512, 16), (18, 7, 3), (34, 65, 33), (1026, 129, 47),
                                     (100, 257, 1), (5000, 64, 80), (3000, 70, 100), (4000, 256, 64),
                                     (3500, 384, 60), (8194, 40, 48)])
def test_sketch_within_contract(engine, spid, m, n, ell):
    """Normal data: within the contract everywhere, and within the
    reference's own fp64 bound gamma_m from m = 1000 rows on."""
    torch.manual_seed(m + n + ell)
    A = torch.randn((3, n, m), dtype=torch.float64, device="cuda")
    _check(engine, spid, A, ell, seed=1234, base=40, gamma=m >= 1000)


def test_sketch_matches_dmma_kernel(engine, spid):
    torch.manual_seed(1)
    A = torch.randn((6, 256, 20000), dtype=torch.float64, device="cuda") * 3.0 + 1.0
    y8 = engine.sketch(A, 48, seed=77, subdomain_base=3)
    _dmma(engine, True)
    try:
        yd = engine.sketch(A, 48, seed=77, subdomain_base=3)
    finally:
        _dmma(engine, False)
    torch.cuda.synchronize()
    for s in range(6):
        om = spid.philox_omega(77, 3 + s, 48, 20000)
        cb, B = _contract(om, _host(A[s]))
        d = np.abs(_host(y8[s]) - _host(yd[s]))
        assert np.all(d <= cb + 2 * _gamma(20000) * B)


@pytest.mark.parametrize("ell", [48, 80])
def test_exponent_changes_and_zero_columns(engine, spid, ell):
    """Columns whose magnitude grows far beyond the first rows' exponent (the
    headroom slow path), all-zero columns, columns zero then nonzero, and
    extreme but finite magnitudes."""
    m, n = 70000, 40
    A = torch.randn((2, n, m), dtype=torch.float64, device="cuda")
    r = torch.arange(m, device="cuda", dtype=torch.float64)
    A[0, 0] *= torch.exp(r / 2000.0)           # grows by e^35 ~ 2^50 over the column
    A[0, 1].zero_()                            # all zero
    A[0, 2, :40000] = 0.0                      # zero, then normal
    A[0, 3] *= 1e300                           # huge
    A[0, 4] *= 1e-290                          # tiny (products stay normal for the oracle)
    A[0, 5, 12345] = 1e6                       # one spike far above the rest
    A[1, 6] = torch.where(r % 2 == 0, 1e-8, 1e4)  # alternating scales
    A[1, 7, ::1000] *= 1e10
    Y, _ = _check(engine, spid, A, ell, seed=3, base=0)
    assert torch.equal(Y[0, 1], torch.zeros_like(Y[0, 1]))


@pytest.mark.parametrize("ell", [48, 80])
def test_adversarial_fixed_point_columns(engine, spid, ell):
    """Columns built against the per-epoch fixed point: an O(1) spike in a
    segment's first stage followed by a long 1e-12 tail in the same segment
    (the tail would be quantised at the spike's scale without the fallback),
    a 1e-12 QoI block after O(1) rows, a single huge row mid-segment then
    tiny rows, a slowly decaying column, and a column whose tail is 2^-30
    of the first stage."""
    m, n = 3 * 4096 + 78, 10
    torch.manual_seed(9)
    A = torch.randn((1, n, m), dtype=torch.float64, device="cuda")
    A[0, 0, 32:4096] *= 1e-12                  # spike stage, then tiny tail (one segment)
    A[0, 1, 5000:] *= 1e-12                    # O(1) rows, then a 1e-12 "QoI block"
    A[0, 2] *= 1e-12
    A[0, 2, 4096 + 100] = 1.0                  # one O(1) row inside tiny rows
    A[0, 3] *= torch.exp(-torch.arange(m, device="cuda", dtype=torch.float64) / 300.0)
    A[0, 4, 16:] *= 2.0 ** -30
    A[0, 5, ::2] = 0.0                         # half zeros
    A[0, 6] = torch.where(torch.arange(m, device="cuda") % 64 < 32, 1.0, 1e-15).double() * A[0, 6]
    _check(engine, spid, A, ell, seed=17, base=2)


def test_nonfinite_poisons_column(engine):
    A = torch.randn((2, 64, 5000), dtype=torch.float64, device="cuda")
    A[0, 5, 4321] = float("nan")
    A[1, 9, 0] = float("inf")
    A[1, 10, 4999] = -float("inf")
    Y = engine.sketch(A, 32, seed=1)
    fin = torch.isfinite(Y)
    assert not fin[0, 5].any() and not fin[1, 9].any() and not fin[1, 10].any()
    fin[0, 5] = True
    fin[1, 9] = True
    fin[1, 10] = True
    assert fin.all()  # other columns untouched


def test_deterministic_and_batch_independent(engine):
    """Bitwise run-to-run stable, and the same subdomain sketched alone, in
    a larger batch at any position, with the grid capped to any SM count or
    run as CTA pairs gives bitwise the same Y (fixed 4096-row segments,
    segment-order reduction)."""
    from paper_2103_01380_b200 import _native as N

    torch.manual_seed(2)
    A = torch.randn((7, 256, 30000), dtype=torch.float64, device="cuda")
    y1 = engine.sketch(A, 48, seed=9)
    y2 = engine.sketch(A, 48, seed=9)
    assert torch.equal(y1, y2)
    for lo, hi in ((3, 4), (2, 5), (0, 4), (3, 7)):
        y3 = engine.sketch(A[lo:hi].contiguous(), 48, seed=9, subdomain_base=lo)
        assert torch.equal(y3, y1[lo:hi]), (lo, hi)
    try:
        for sms in (1, 5, 37, 132):
            engine.h.check(N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_SKETCH_SMS, sms))
            assert torch.equal(engine.sketch(A, 48, seed=9), y1), sms
    finally:
        engine.h.check(N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_SKETCH_SMS, 0))
    for mode in (0, 2):
        _pairs(engine, mode)
        assert torch.equal(engine.sketch(A, 48, seed=9), y1), mode
    _pairs(engine, 1)


@pytest.mark.parametrize("ell", [30, 64, 80])
def test_batch_independent_all_widths(engine, ell):
    """Every pass width (one pass, a 64-row pass, two passes for ell = 80)
    and the DMMA kernel (explicit-Omega oracle mode) alike."""
    torch.manual_seed(ell)
    A = torch.randn((5, 256, 9000), dtype=torch.float64, device="cuda")
    y = engine.sketch(A, ell, seed=4)
    for lo in range(5):
        assert torch.equal(engine.sketch(A[lo:lo + 1].contiguous(), ell, seed=4, subdomain_base=lo), y[lo:lo + 1])
    _dmma(engine, True)
    try:
        yd = engine.sketch(A, ell, seed=4)
        assert torch.equal(engine.sketch(A[1:3].contiguous(), ell, seed=4, subdomain_base=1), yd[1:3])
    finally:
        _dmma(engine, False)


@pytest.mark.parametrize("sms", [1, 37, 132])
def test_sketch_sm_cap(engine, spid, sms):
    """SPIDGPU_OPT_SKETCH_SMS: a persistent grid capped to fewer SMs still
    meets the bound, and resets to all SMs."""
    from paper_2103_01380_b200 import _native as N

    torch.manual_seed(5)
    A = torch.randn((3, 200, 9000), dtype=torch.float64, device="cuda")
    try:
        engine.h.check(N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_SKETCH_SMS, sms))
        _check(engine, spid, A, 40, 21, 0)
    finally:
        engine.h.check(N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_SKETCH_SMS, 0))
    assert N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_SKETCH_SMS, -1) != 0
    for bad in (-1, 3):
        assert N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_SKETCH_PAIRS, bad) != 0
    assert N.lib.spidgpu_set_option(engine.h.h, 3, 1) != 0  # the retired IMMA option


def test_large_subdomain_cfg3_shape(engine, spid):
    """One config-3 subdomain (163840 x 256, 40 segments), against the oracle
    within 2 gamma_m (the extended-precision product is too slow here)."""
    from paper_2103_01380_b200.configs import CONFIGS

    cfg = CONFIGS["cfg3"]
    A = engine.generate(cfg, 5, 1)
    _check(engine, spid, A, cfg.ell, seed=cfg.seed, base=5, exact=False)


def test_large_subdomain_cfg4_shape(engine, spid):
    """One config-4 heavy subdomain (163840 x 256, +256 high-wavenumber
    modes), ell = 80 in one pass (slice-split CTA pairs, 20 segments of 8192
    rows, two partials each), against the oracle's fp64 matmul within the
    contract + gamma_m; and bitwise the same Y when sketched inside a batch
    of four."""
    import numpy as np

    from paper_2103_01380_b200.configs import CONFIGS

    cfg = CONFIGS["cfg4"]
    heavy = np.array([0, 1, 1, 0], dtype=np.uint8)
    A = engine.generate(cfg, 0, 4, heavy=heavy)
    Y1, _ = _check(engine, spid, A[1:2].contiguous(), cfg.ell, seed=cfg.seed, base=1, exact=False)
    Y4 = engine.sketch(A, cfg.ell, seed=cfg.seed, subdomain_base=0)
    assert torch.equal(Y4[1:2], Y1)


def test_padded_leading_dimension_and_stride(engine, spid):
    """lda > m and strideA > lda*n (a padded, strided batch) through the C ABI:
    the TMA tensor map walks the strides, padding rows are never read."""
    import ctypes as C

    from paper_2103_01380_b200 import _native as N

    m, n, S, ell, lda = 3000, 150, 3, 48, 3010
    stride = lda * n + 64
    torch.manual_seed(11)
    buf = torch.full((S * stride,), float("nan"), dtype=torch.float64, device="cuda")
    dense = torch.randn((S, n, m), dtype=torch.float64, device="cuda")
    for s in range(S):
        view = buf[s * stride: s * stride + lda * n].view(n, lda)
        view[:, :m] = dense[s]
    Y = torch.empty((S, n, ell), dtype=torch.float64, device="cuda")
    om = engine.omega(21, 7)
    engine.h.check(N.lib.spidgpu_sketch_batched(engine.h.h, C.c_void_p(buf.data_ptr()), m, n, lda, stride,
                                                S, ell, C.byref(om), C.c_void_p(Y.data_ptr()), ell, ell * n,
                                                None))
    torch.cuda.synchronize()
    assert torch.isfinite(Y).all()  # the NaN padding was never contracted
    assert torch.equal(Y, engine.sketch(dense, ell, seed=21, subdomain_base=7))
    for s in range(S):
        _bound_check(_host(Y[s]), spid.philox_omega(21, 7 + s, ell, m), _host(dense[s]))
