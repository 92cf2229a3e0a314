"""GPU Gaussian-sketch path (sketch -> CPQR -> gather -> verify) against the
CPU oracle, in oracle mode (explicit Omega) and in performance mode (in-kernel
Philox Omega, materialised with spidgpu_philox_omega for the oracle).

Tolerances (north_star): Y to 1e-13 relative (reordered fp64
summation); pivots bit-exact except documented near ties (tests/parity.py);
coefficients within tol_C = max(1e-10, 1e3 eps kappa_hat); relative
reconstruction error within 1e-3 relative."""
import numpy as np
import pytest
import torch

from parity import ERR_RTOL, compare_pivots, rel_maxdiff, tol_coeffs

pytestmark = pytest.mark.gpu


def _host(t):
    """(n, m) row-major device tensor -> (m, n) Fortran numpy (same bytes)."""
    return np.asfortranarray(t.detach().cpu().numpy().T)


def _check_subdomain(orc, a, omega, k, y_gpu, idx_gpu, c_gpu, resid_gpu, err2_gpu=None,
                     ref2_gpu=None):
    o = orc.sketch_id(a, omega, rank=k)
    # Y: reordered-summation fp64 agreement, per column relative to its norm
    scale = np.linalg.norm(o.y, axis=0)
    dy = np.max(np.abs(y_gpu - o.y) / np.maximum(scale, 1e-300))
    assert dy <= 1e-13, dy
    s, ok, gap = compare_pivots(o.y, idx_gpu, o.indices)
    assert ok, f"pivot divergence at step {s} with gap {gap}"
    qr = orc.qr(o.y, rank=k)
    diag = np.abs(np.diag(qr.r[:, :k]))
    tc = tol_coeffs(diag)
    assert rel_maxdiff(c_gpu, o.coeffs) <= tc
    assert abs(resid_gpu - o.residual_fro) <= 1e-6 * max(o.residual_fro, 1e-300) + 1e-12 * np.linalg.norm(o.y)
    if err2_gpu is not None:
        e2, r2 = orc.error_terms(a, o.skeleton, o.coeffs)
        assert abs(np.sqrt(err2_gpu / ref2_gpu) - np.sqrt(e2 / r2)) <= ERR_RTOL * np.sqrt(e2 / r2)
        assert abs(ref2_gpu - r2) <= 1e-12 * r2
    return o


@pytest.mark.parametrize("m,n,ell,k", [(16384, 100, 20, 10), (4096, 256, 48, 32),
                                       (1000, 37, 30, 20), (2048, 512, 30, 20),
                                       (5000, 256, 80, 64), (3000, 64, 100, 40)])
def test_sketch_explicit_omega_matches_matmul(engine, orc, m, n, ell, k):
    torch.manual_seed(0)
    A = torch.randn((2, n, m), dtype=torch.float64, device="cuda")
    omegas = [orc.gaussian(ell, m, 100 + s) for s in range(2)]
    om_t = torch.stack([torch.from_numpy(np.ascontiguousarray(o.T)) for o in omegas]).cuda()
    Y = engine.sketch(A, ell, omega=om_t)
    torch.cuda.synchronize()
    for s in range(2):
        y_ref = orc.matmul(omegas[s], _host(A[s]))
        y = _host(Y[s])
        scale = np.linalg.norm(y_ref, axis=0)
        assert np.max(np.abs(y - y_ref) / scale) <= 1e-13


def test_sketch_philox_matches_materialised_omega(engine, spid, orc):
    m, n, ell = 6000, 130, 48
    A = torch.randn((3, n, m), dtype=torch.float64, device="cuda")
    Y = engine.sketch(A, ell, seed=1234, subdomain_base=40)
    for s in range(3):
        om = spid.philox_omega(1234, 40 + s, ell, m)
        # Gaussian moments of the generator (discretised N(0,1), Q/32)
        assert abs(om.mean()) < 0.02 and abs(om.std() - 1.0) < 0.02
        y_ref = orc.matmul(om, _host(A[s]))
        scale = np.linalg.norm(y_ref, axis=0)
        assert np.max(np.abs(_host(Y[s]) - y_ref) / scale) <= 1e-13


def test_sketch_ragged_and_oob(engine, orc):
    # m not a multiple of the 16-row chunk, n not a multiple of the column tile
    for m, n in [(18, 7), (34, 65), (1026, 129), (100, 257)]:
        A = torch.randn((3, n, m), dtype=torch.float64, device="cuda")
        om = [orc.gaussian(12, m, s) for s in range(3)]
        om_t = torch.stack([torch.from_numpy(np.ascontiguousarray(o.T)) for o in om]).cuda()
        Y = engine.sketch(A, 12, omega=om_t)
        for s in range(3):
            y_ref = orc.matmul(om[s], _host(A[s]))
            assert rel_maxdiff(_host(Y[s]), y_ref) <= 1e-13


def test_cpqr_on_oracle_sketch_is_bitwise(engine, orc):
    """Same Y in -> identical pivots, C, residual (the CPQR restates the
    reference's exact operation order)."""
    from paper_2103_01380_b200.spid import RankRule

    rng = np.random.default_rng(0)
    ys = [orc.matmul(orc.gaussian(48, 500, 7 + s), orc.seeded_matrix(500, 256, 70 + s)) for s in range(4)]
    Y = torch.stack([torch.from_numpy(np.ascontiguousarray(y.T)) for y in ys]).cuda()
    res = engine.cpqr(Y, RankRule.fixed(32))
    res.check()
    for s, y in enumerate(ys):
        o = orc.column_id(y, rank=32)
        assert np.array_equal(res.indices[s].cpu().numpy(), o.indices)
        c = np.asfortranarray(res.coeffs[s].cpu().numpy().T)
        assert np.array_equal(c, o.coeffs)
        assert float(res.residual_fro[s]) == o.residual_fro
    _ = rng


def test_cfg1_end_to_end(engine, spid, orc):
    """BASELINE config 1 (the reference's CPU-runnable case): TGV 32^3, 4 QoIs,
    100 snapshots, 8 subdomains of 16^3, k=10, p=10, Philox Omega."""
    from paper_2103_01380_b200.configs import CONFIGS
    from paper_2103_01380_b200.engine import rule_for

    cfg = CONFIGS["cfg1"]
    A = engine.generate(cfg, 0, cfg.subdomains)
    r = engine.compress(A, cfg.ell, rule_for(cfg), seed=cfg.seed, want_sketch=True)
    r.check()
    err2, ref2 = engine.verify(A, r)
    torch.cuda.synchronize()
    tot_e = tot_r = 0.0
    for s in range(cfg.subdomains):
        a = _host(A[s])
        om = spid.philox_omega(cfg.seed, s, cfg.ell, cfg.m)
        c = np.asfortranarray(r.coeffs[s].cpu().numpy().T)
        o = _check_subdomain(orc, a, om, cfg.k, _host(r.sketch[s]), r.indices[s].cpu().numpy(), c,
                             float(r.residual_fro[s]), float(err2[s]), float(ref2[s]))
        # skeleton gather is a bit-exact copy of A(:, I)
        skel = np.asfortranarray(r.skel[s].cpu().numpy().T)
        assert np.array_equal(skel, a[:, r.indices[s].cpu().numpy()])
        e2, r2 = orc.error_terms(a, o.skeleton, o.coeffs)
        tot_e += e2
        tot_r += r2
    rel = np.sqrt(err2.sum().item() / ref2.sum().item())
    assert abs(rel - np.sqrt(tot_e / tot_r)) <= ERR_RTOL * np.sqrt(tot_e / tot_r)
    cf = spid.compression_factor(cfg.m * cfg.subdomains, cfg.n,
                                 int(r.stored_entries().sum().item()))
    assert abs(cf - 9.94) < 0.01  # 16384*100 / (10*(16384+100))
    assert rel < 1e-6


def test_determinism_bitwise(engine):
    from paper_2103_01380_b200.spid import RankRule

    A = torch.randn((5, 256, 8192), dtype=torch.float64, device="cuda")
    r1 = engine.compress(A, 48, RankRule.fixed(32), seed=9, want_sketch=True)
    r2 = engine.compress(A, 48, RankRule.fixed(32), seed=9, want_sketch=True)
    assert torch.equal(r1.sketch, r2.sketch)
    assert torch.equal(r1.coeffs, r2.coeffs) and torch.equal(r1.indices, r2.indices)
    e1 = engine.verify(A, r1)
    e2 = engine.verify(A, r2)
    assert torch.equal(e1[0], e2[0]) and torch.equal(e1[1], e2[1])


def test_batch_status_isolation(engine):
    """A failing subdomain reports its own reference error name; the others
    still compress (per-subdomain status array)."""
    from paper_2103_01380_b200.spid import RankRule

    A = torch.randn((4, 64, 1000), dtype=torch.float64, device="cuda")
    A[1, 3, 17] = float("nan")
    A[2].zero_()
    r = engine.compress(A, 20, RankRule.fixed(8), seed=1)
    st = r.status.cpu().tolist()
    assert st[0] == 0 and st[3] == 0
    assert st[1] == 1  # NonFiniteInput
    assert st[2] == 3  # ZeroMatrix


def test_sketch_id_host_api(spid, orc):
    a = orc.seeded_matrix(3001, 90, 17)
    om = orc.gaussian(24, 3001, 18)
    g = spid.sketch_id(a, 24, rank=12, omega=om, want_sketch=True)
    o = orc.sketch_id(a, om, rank=12)
    assert rel_maxdiff(g.sketch, o.y) <= 1e-13
    s, ok, _ = compare_pivots(o.y, g.skeleton_indices, o.indices)
    assert ok
    assert np.array_equal(g.skeleton, a[:, g.skeleton_indices])
