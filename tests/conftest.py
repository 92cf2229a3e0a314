import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libspidgpu.so")


@pytest.fixture(scope="session")
def orc():
    import oracle

    return oracle.port()


@pytest.fixture(scope="session")
def ref():
    import oracle

    if not oracle.ref_available():
        pytest.skip("oracle/_ref (reference compiled from /root/reference) not built")
    return oracle.ref()


@pytest.fixture(scope="session")
def spid():
    from paper_2103_01380_b200 import spid as s

    return s


@pytest.fixture(scope="session")
def engine():
    from paper_2103_01380_b200.engine import Engine

    return Engine(0)


def tgv2d(dims=(20, 20), steps=100, dt=0.1, nu=0.1, rho=1.0, qoi="u1"):
    """2D analytic Taylor-Green snapshot matrix, restating
    proj/src/datagen.cpp:47-80 (x_i = 2*pi*i/N, axis 0 fastest)."""
    n0, n1 = dims
    i = np.arange(n0 * n1)
    x = 2 * np.pi * (i % n0) / n0
    y = 2 * np.pi * ((i // n0) % n1) / n1
    cols = []
    for j in range(steps):
        t = dt * j
        d2, d4 = np.exp(-2 * nu * t), np.exp(-4 * nu * t)
        if qoi == "u1":
            c = np.sin(x) * np.cos(y) * d2
        elif qoi == "u2":
            c = -np.cos(x) * np.sin(y) * d2
        else:
            c = 0.25 * rho * (np.cos(2 * x) + np.sin(2 * y)) * d4
        cols.append(c)
    return np.asfortranarray(np.stack(cols, axis=1))
