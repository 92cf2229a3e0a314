"""The CPU workload generator of the reference arm (oracle/workload.c):
Omega's quantile table and Philox stream, and the BASELINE synthetic fields,
checked against the product's definitions -- so `bench.py --impl reference`
times the same workload without loading libspidgpu.so."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _product_table():
    src = open(os.path.join(ROOT, "paper_2103_01380_b200", "csrc", "omega_table.h")).read()
    body = src[src.index("SPIDGPU_OMEGA_TABLE_INIT"):]
    return np.array([int(v) for v in re.findall(r"-?\d+", body[body.index("{"):body.index("}")])],
                    dtype=np.int8)


def test_omega_table_matches_product(orc):
    q = orc.omega_table()
    assert np.array_equal(q, _product_table())
    assert np.all(q == -q[::-1]) and np.abs(q).max() == 117


def test_philox_omega_statistics_and_counter(orc):
    om = orc.philox_omega(5, 3, 48, 20000)
    q = om * 32
    assert np.array_equal(q, np.rint(q)) and np.abs(q).max() <= 117
    assert abs(om.mean()) < 0.01 and abs(om.std() - 1.0) < 0.01
    # rows are independent counters: a row slice equals the full matrix's rows
    assert np.array_equal(orc.philox_omega(5, 3, 16, 20000, row0=32), om[32:48])
    assert not np.array_equal(orc.philox_omega(5, 4, 48, 20000), om)


def test_tgv4_field_formula(orc):
    """Config 1 (analytic TGV, no noise): spot values of u, v, w, p against
    the BASELINE formulas with x_i = 2 pi i / N (proj/src/datagen.cpp:26)."""
    from paper_2103_01380_b200.configs import CONFIGS

    cfg = CONFIGS["cfg1"]
    spec = dict(cfg.field_dict(), sigma=0.0)
    a = orc.field_generate(spec, 3, 1, threads=2)[0]  # (n, m)
    b, N = cfg.block, cfg.grid
    nb = N // b
    g = 3
    bx, by, bz = g % nb, (g // nb) % nb, g // (nb * nb)
    for pt in (0, 5, 100, b ** 3 - 1):
        ix, iy, iz = bx * b + pt % b, by * b + (pt // b) % b, bz * b + pt // (b * b)
        x, y, z = (2 * np.pi * i / N for i in (ix, iy, iz))
        for j in (0, 37, 99):
            t = cfg.t_end * j / (cfg.n - 1)
            F = np.exp(-2 * cfg.nu * t)
            u = np.sin(x) * np.cos(y) * np.cos(z) * F
            v = -np.cos(x) * np.sin(y) * np.cos(z) * F
            p = (np.cos(2 * x) + np.cos(2 * y)) * (np.cos(2 * z) + 2) * F * F / 16
            got = [a[j, q * b ** 3 + pt] for q in range(4)]
            np.testing.assert_allclose(got, [u, v, 0.0, p], rtol=1e-14, atol=1e-15)


def test_field_generate_threads_and_ranges(orc):
    from paper_2103_01380_b200.configs import CONFIGS

    cfg = CONFIGS["cfg2"]
    spec = dict(cfg.field_dict(), snapshots=8)
    a1 = orc.field_generate(spec, 10, 3, threads=1)
    a4 = orc.field_generate(spec, 10, 3, threads=4)
    assert np.array_equal(a1, a4)  # thread count does not change the bits
    assert np.array_equal(orc.field_generate(spec, 11, 1, threads=3)[0], a1[1])
    # rho = 1 + 0.01 p and noise ~ sigma
    rho = a1[:, :, :b3(cfg)]
    assert np.all(np.abs(rho - 1) < 0.01)


def b3(cfg):
    return cfg.block ** 3


@pytest.mark.gpu
def test_cpu_workload_matches_device(orc, engine):
    """The device generator and the CPU one describe the same field (libm vs
    device transcendentals: ~1e-15 relative; the fp32 Box-Muller noise to
    its own rounding), and the same Omega bit for bit."""
    import torch

    from paper_2103_01380_b200 import spid
    from paper_2103_01380_b200.configs import CONFIGS

    for name in ("cfg1", "cfg2", "cfg5"):
        cfg = CONFIGS[name]
        spec = cfg.field_dict()
        dev = engine.generate(cfg, 2, 2).cpu().numpy()
        cpu = orc.field_generate(spec, 2, 2)
        scale = np.abs(dev).max()
        # the device draws the fp32 Box-Muller noise with fast intrinsics (__logf,
        # __sincosf): the noise agrees to ~1e-4 of sigma, the field to 1e-12
        assert np.max(np.abs(dev - cpu)) <= 1e-12 * scale + 1e-3 * cfg.sigma, name
    heavy = np.array([1, 0], dtype=np.uint8)
    cfg = CONFIGS["cfg4"]
    dev = engine.generate(cfg, 100, 2, heavy=heavy).cpu().numpy()
    cpu = orc.field_generate(cfg.field_dict(), 100, 2, is_heavy=heavy)
    assert np.max(np.abs(dev - cpu)) <= 1e-12 * np.abs(dev).max()
    for s, ell, m in ((0, 48, 5000), (7, 80, 1234), (2 ** 33 + 5, 3, 64)):
        assert np.array_equal(orc.philox_omega(99, s, ell, m), spid.philox_omega(99, s, ell, m))
    torch.cuda.synchronize()
