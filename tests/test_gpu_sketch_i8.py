"""The exact integer-sliced sketch, which runs every Philox-Omega sketch:
Y = Omega A with Omega = Q/32 integer-valued, A split into 7 byte slices of a
55-bit per-column fixed point, each slice contracted exactly in int32 --
on tcgen05.mma kind::i8 with TMEM accumulators (csrc/sketch_tc.cu, the
default; also forced into its CTA-pair mode, which shares each stage's Omega
tile between the two CTAs of a cluster) and on register-fed IMMA.16832
(csrc/sketch_i8.cu, SPIDGPU_OPT_IMMA_SKETCH). Every test runs on all three.

Checked against the oracle's matmul (proj/src/dense_matrix.cpp:38-53) on the
materialised Omega, and against the FP64 DMMA kernel (SPIDGPU_OPT_DMMA_SKETCH)
on the same Omega. Tolerance: 1e-13 relative per column (north_star's
reordered-fp64 bound), the column scale being sqrt(ell) |A(:,j)| (the
expected norm of a sketch column; a single-row sketch can cancel to far
below it, where both sides' rounding is relative to the terms, not the sum)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _host(t):
    return np.asfortranarray(t.detach().cpu().numpy().T)


def _dmma(engine, on):
    from paper_2103_01380_b200 import _native as N

    engine.h.check(N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_DMMA_SKETCH, int(on)))


@pytest.fixture(params=["tc", "tc_pairs", "imma"], autouse=True)
def kernel(request, engine):
    """Route the Philox sketches of the shared engine to one kernel: tcgen05
    (CTA pairs only for 64-row passes, the default), tcgen05 with CTA pairs
    wherever the column tiles pair up, or register-fed IMMA."""
    from paper_2103_01380_b200 import _native as N

    engine.h.check(N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_IMMA_SKETCH,
                                            int(request.param == "imma")))
    engine.h.check(N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_SKETCH_PAIRS,
                                            2 if request.param == "tc_pairs" else 1))
    yield request.param
    engine.h.check(N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_IMMA_SKETCH, 0))
    engine.h.check(N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_SKETCH_PAIRS, 1))


def _check_vs_oracle(engine, spid, orc, A, ell, seed, base, tol=1e-13):
    Y = engine.sketch(A, ell, seed=seed, subdomain_base=base)
    torch.cuda.synchronize()
    S, n, m = A.shape
    worst = 0.0
    for s in range(S):
        om = spid.philox_omega(seed, base + s, ell, m)
        y_ref = orc.matmul(om, _host(A[s]))
        # natural scale of a sketch column: E|Y(:,j)|^2 = ell |A(:,j)|^2
        a = _host(A[s])
        amax = np.maximum(np.abs(a).max(axis=0), 1e-300)  # overflow-safe norms
        scale = np.sqrt(ell) * amax * np.linalg.norm(a / amax, axis=0)
        scale = np.where(scale > 0, scale, 1.0)
        d = np.max(np.abs(_host(Y[s]) - y_ref) / scale)
        worst = max(worst, d)
    assert worst <= tol, worst
    return Y


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
                                     (3500, 384, 60)])
def test_i8_sketch_matches_oracle(engine, spid, orc, m, n, ell):
    torch.manual_seed(m + n + ell)
    A = torch.randn((3, n, m), dtype=torch.float64, device="cuda")
    _check_vs_oracle(engine, spid, orc, A, ell, seed=1234, base=40)


def test_i8_matches_dmma_kernel(engine):
    torch.manual_seed(1)
    A = torch.randn((6, 256, 20000), dtype=torch.float64, device="cuda") * 3.0 + 1.0
    y8 = engine.sketch(A, 48, seed=77, subdomain_base=3)
    _dmma(engine, True)
    try:
        yd = engine.sketch(A, 48, seed=77, subdomain_base=3)
    finally:
        _dmma(engine, False)
    scale = yd.norm(dim=2, keepdim=True)
    assert ((y8 - yd).abs() / scale).max().item() <= 1e-13


def test_i8_exponent_changes_and_zero_columns(engine, spid, orc):
    """Columns whose magnitude grows far beyond the first rows' exponent (the
    headroom slow path), all-zero columns, columns zero then nonzero, and
    extreme but finite magnitudes."""
    m, n = 70000, 40  # > 65536 rows: one int32 flush period boundary inside
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
    _check_vs_oracle(engine, spid, orc, A, 48, seed=3, base=0)


def test_i8_nonfinite_poisons_column(engine):
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


def test_i8_deterministic_and_partition_independent(engine):
    """Bitwise run-to-run stable; the same subdomain sketched alone or inside
    a larger batch (different stream-K split, so different fixed-point
    periods and exponents) agrees to the fixed-point rounding (2^-47 of the
    period's scale for the tcgen05 kernel's 50-bit fixed point)."""
    torch.manual_seed(2)
    A = torch.randn((7, 256, 30000), dtype=torch.float64, device="cuda")
    y1 = engine.sketch(A, 48, seed=9)
    y2 = engine.sketch(A, 48, seed=9)
    assert torch.equal(y1, y2)
    y3 = engine.sketch(A[3:4].contiguous(), 48, seed=9, subdomain_base=3)
    scale = y1[3].norm(dim=1, keepdim=True)
    assert ((y3[0] - y1[3]).abs() / scale).max().item() <= 1e-14


@pytest.mark.parametrize("sms", [1, 37, 132])
def test_i8_sketch_sm_cap(engine, spid, orc, sms):
    """SPIDGPU_OPT_SKETCH_SMS: a persistent grid capped to fewer SMs (other
    stream-K splits) still matches the oracle, and resets to all SMs."""
    from paper_2103_01380_b200 import _native as N

    torch.manual_seed(5)
    A = torch.randn((3, 200, 9000), dtype=torch.float64, device="cuda")
    try:
        engine.h.check(N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_SKETCH_SMS, sms))
        _check_vs_oracle(engine, spid, orc, A, 40, 21, 0)
    finally:
        engine.h.check(N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_SKETCH_SMS, 0))
    assert N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_SKETCH_SMS, -1) != 0
    for bad in (-1, 3):
        assert N.lib.spidgpu_set_option(engine.h.h, N.SPIDGPU_OPT_SKETCH_PAIRS, bad) != 0


def test_i8_large_subdomain_cfg3_shape(engine, spid, orc):
    """One config-3 subdomain (163840 x 256, three flush periods)."""
    from paper_2103_01380_b200.configs import CONFIGS

    cfg = CONFIGS["cfg3"]
    A = engine.generate(cfg, 5, 1)
    _check_vs_oracle(engine, spid, orc, A, cfg.ell, seed=cfg.seed, base=5)


def test_i8_padded_leading_dimension_and_stride(engine, spid, orc):
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
    for s in range(S):
        o = spid.philox_omega(21, 7 + s, ell, m)
        y_ref = orc.matmul(o, _host(dense[s]))
        a = _host(dense[s])
        scale = np.sqrt(ell) * np.linalg.norm(a, axis=0)
        assert np.max(np.abs(_host(Y[s]) - y_ref) / scale) <= 1e-13
