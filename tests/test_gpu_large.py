"""GPU checks at BASELINE.json's full subdomain sizes (163840 x 256 / 512 fp64),
where the CPU oracle would take minutes per subdomain: size-independent
properties plus a plain-torch fp64 reference for the floating-point kernels.

* gather: skel == A(:, I) bit for bit;
* coefficients: exact identity block C(:, I) = I (proj/src/id.cpp:12);
* residual identity on the sketch: ||Y - Y(:, I) C||_F == residual_fro
  (acceptance.cpp:325-344, here for Y);
* sketch linearity: sketch(A1 + A2) == sketch(A1) + sketch(A2) (fp64 rel. 1e-12);
* verify: err2/ref2 vs torch fp64 (bmm) to 1e-9 relative;
* determinism: two runs bitwise equal;
* one full subdomain per config is also checked against the CPU oracle with
  the materialised Philox Omega."""
import numpy as np
import pytest
import torch

from parity import ERR_RTOL, compare_pivots, rel_maxdiff, tol_coeffs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg3_batch(engine):
    from paper_2103_01380_b200.configs import CONFIGS

    cfg = CONFIGS["cfg3"]
    field = CONFIGS["cfg5"]
    A = engine.generate(field, 0, 6)
    return cfg, A


def _host(t):
    return np.asfortranarray(t.detach().cpu().numpy().T)


def test_cfg3_properties(engine, cfg3_batch):
    from paper_2103_01380_b200.engine import rule_for

    cfg, A = cfg3_batch
    r = engine.compress(A, cfg.ell, rule_for(cfg), seed=cfg.seed, want_sketch=True)
    r.check()
    S, n, m = A.shape
    idx = r.indices
    for s in range(S):
        k = int(r.rank[s])
        assert k == cfg.k
        # gather is a bit-exact copy
        assert torch.equal(r.skel[s, :k], A[s, idx[s, :k]])
        # identity block, exactly
        C = r.coeffs[s, :, :k].T  # k x n
        assert torch.equal(C[:, idx[s, :k]], torch.eye(k, dtype=torch.float64, device=A.device))
        # residual identity on the sketch
        Y = r.sketch[s].T  # ell x n
        res = torch.linalg.norm(Y - Y[:, idx[s, :k]] @ C)
        assert abs(res.item() - float(r.residual_fro[s])) <= 1e-9 * float(r.residual_fro[s]) + \
            1e-14 * torch.linalg.norm(Y).item()


def test_verify_vs_torch_fp64(engine, cfg3_batch):
    from paper_2103_01380_b200.engine import rule_for

    cfg, A = cfg3_batch
    r = engine.compress(A, cfg.ell, rule_for(cfg), seed=cfg.seed)
    err2, ref2 = engine.verify(A, r)
    for s in range(A.shape[0]):
        k = int(r.rank[s])
        Sk = r.skel[s, :k].T            # m x k
        C = r.coeffs[s, :, :k].T        # k x n
        Aref = A[s].T                   # m x n
        e2 = torch.linalg.norm(Aref - Sk @ C).item() ** 2
        r2 = torch.linalg.norm(Aref).item() ** 2
        assert abs(err2[s].item() - e2) <= 1e-9 * e2
        assert abs(ref2[s].item() - r2) <= 1e-12 * r2


def test_sketch_linearity(engine, cfg3_batch):
    cfg, A = cfg3_batch
    A1 = A[:2].clone()
    A2 = torch.randn_like(A1)
    y1 = engine.sketch(A1, cfg.ell, seed=5)
    y2 = engine.sketch(A2, cfg.ell, seed=5)
    y12 = engine.sketch(A1 + A2, cfg.ell, seed=5)
    scale = torch.linalg.norm(y12, dim=2, keepdim=True)
    assert ((y12 - y1 - y2).abs() / scale).max().item() <= 1e-12


def test_full_subdomain_vs_oracle(engine, spid, orc, cfg3_batch):
    """One 163840 x 256 subdomain end to end against the CPU oracle fed the
    same Philox Omega (SURVEY 8(c) parity protocol)."""
    from paper_2103_01380_b200.engine import rule_for

    cfg, A = cfg3_batch
    s = 3
    r = engine.compress(A[s:s + 1], cfg.ell, rule_for(cfg), seed=cfg.seed, subdomain_base=s,
                        want_sketch=True)
    err2, ref2 = engine.verify(A[s:s + 1], r)
    a = _host(A[s])
    om = spid.philox_omega(cfg.seed, s, cfg.ell, cfg.m)
    o = orc.sketch_id(a, om, rank=cfg.k)
    y = _host(r.sketch[0])
    assert rel_maxdiff(y, o.y) <= 1e-12
    step, ok, gap = compare_pivots(o.y, r.indices[0].cpu().numpy(), o.indices)
    assert ok, (step, gap)
    if step == cfg.k:  # identical selection -> coefficient tolerance applies
        q = orc.qr(o.y, rank=cfg.k)
        tc = tol_coeffs(np.abs(np.diag(q.r[:, :cfg.k])))
        c = np.asfortranarray(r.coeffs[0].cpu().numpy().T)
        assert rel_maxdiff(c, o.coeffs) <= tc
    e2, r2 = orc.error_terms(a, o.skeleton, o.coeffs)
    rel_gpu = np.sqrt(err2[0].item() / ref2[0].item())
    rel_orc = np.sqrt(e2 / r2)
    assert abs(rel_gpu - rel_orc) <= ERR_RTOL * rel_orc


def test_cfg2_shape_vs_oracle(engine, spid, orc):
    """Config 2 shape (163840 x 512, ell = 30, k = 20): one subdomain."""
    from paper_2103_01380_b200.configs import CONFIGS
    from paper_2103_01380_b200.engine import rule_for

    cfg = CONFIGS["cfg2"]
    A = engine.generate(cfg, 5, 1)
    r = engine.compress(A, cfg.ell, rule_for(cfg), seed=cfg.seed, subdomain_base=5,
                        want_sketch=True)
    r.check()
    err2, ref2 = engine.verify(A, r)
    a = _host(A[0])
    om = spid.philox_omega(cfg.seed, 5, cfg.ell, cfg.m)
    o = orc.sketch_id(a, om, rank=cfg.k)
    assert rel_maxdiff(_host(r.sketch[0]), o.y) <= 1e-12
    step, ok, gap = compare_pivots(o.y, r.indices[0].cpu().numpy(), o.indices)
    assert ok, (step, gap)
    e2, r2 = orc.error_terms(a, o.skeleton, o.coeffs)
    assert abs(np.sqrt(err2[0].item() / ref2[0].item()) - np.sqrt(e2 / r2)) <= ERR_RTOL * np.sqrt(e2 / r2)


def test_cfg4_blocked_rank_rule(engine, orc):
    """Config 4: rank grows in steps of 8 up to 64 until the sketch error
    <= 1e-3; heavy subdomains (extra high-wavenumber modes) need more rank.
    Blocked-rule CPQR on the GPU sketch equals the oracle's bit for bit."""
    from paper_2103_01380_b200.configs import CONFIGS
    from paper_2103_01380_b200.engine import rule_for

    cfg = CONFIGS["cfg4"]
    heavy = np.array([0, 1, 0, 1], dtype=np.uint8)
    A = engine.generate(cfg, 0, 4, heavy=heavy)
    r = engine.compress(A, cfg.ell, rule_for(cfg), seed=cfg.seed, want_sketch=True)
    r.check()
    ranks = r.rank.cpu().numpy()
    assert all(k % 8 == 0 and 8 <= k <= 64 for k in ranks)
    for s in range(4):
        y = _host(r.sketch[s])
        o = orc.column_id(y, rank=cfg.k, tol=cfg.tol, kstep=cfg.kstep)
        assert o.rank == ranks[s]
        assert np.array_equal(o.indices, r.indices[s, :o.rank].cpu().numpy())
        assert o.residual_fro <= cfg.tol * np.linalg.norm(y) or o.rank == 64
    assert ranks[1] >= ranks[0] and ranks[3] >= ranks[2]


def test_compress_host_matches_device(engine, cfg3_batch):
    """spidgpu_compress_host (host buffers, copies inside, groups of g
    subdomains) == the device path over the whole batch, bitwise, for any
    group size: sketch, CPQR, gather and verify do not depend on how the
    subdomains are batched (fixed 4096-row segments, fixed-order sums)."""
    from paper_2103_01380_b200.engine import rule_for

    cfg, A = cfg3_batch
    rule = rule_for(cfg)
    r = engine.compress(A[:5], cfg.ell, rule, seed=cfg.seed, subdomain_base=0)
    err2, ref2 = engine.verify(A[:5], r)
    a_host = A[:5].cpu().pin_memory()
    for g in (1, 2, 3, 8):
        out = engine.compress_host(a_host, cfg.ell, rule, seed=cfg.seed, group=g, verify=True)
        assert torch.equal(out["indices"], r.indices.cpu()), g
        assert torch.equal(out["coeffs"], r.coeffs.cpu()), g
        assert torch.equal(out["skel"], r.skel.cpu()), g
        assert torch.equal(out["err2"], err2.cpu()), g
        assert torch.equal(out["ref2"], ref2.cpu()), g
