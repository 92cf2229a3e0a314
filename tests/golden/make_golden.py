"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref, compiled
from /root/reference/proj/src by oracle/Makefile). Run here, where
/root/reference exists; the fixtures are committed so the CPU tests (and the
GPU box, which has no /root/reference) can pin the oracle against them.

    python tests/golden/make_golden.py
"""
import os
import sys

import hashlib

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def digest(a: np.ndarray) -> np.ndarray:
    """Inputs are regenerated from their SplitMix64 seeds by the tests; the
    fixture stores a SHA-256 of the column-major bytes to pin them."""
    h = hashlib.sha256(np.asfortranarray(a).tobytes(order="F")).digest()
    return np.frombuffer(h, dtype=np.uint8).copy()


def main():
    ref = oracle.ref()
    port = oracle.port()
    cases = {}
    # column_id / qr on SplitMix64-seeded matrices (proj/tests/common.hpp:13-19)
    shapes = [(3, 3), (7, 2), (9, 6), (14, 9), (15, 10), (16, 11), (20, 12), (33, 17),
              (48, 64), (30, 40), (5, 12)]
    for si, (m, n) in enumerate(shapes):
        seed = 4000 + si
        a = port.seeded_matrix(m, n, seed)
        for k in sorted({1, min(3, m, n), min(m, n)}):
            f = ref.column_id(a, rank=k)
            q = ref.qr(a, rank=k)
            key = f"cid_{m}x{n}_k{k}"
            cases[key + "_seed"] = np.array([seed, m, n, k], dtype=np.int64)
            cases[key + "_a_sha"] = digest(a)
            cases[key + "_indices"] = f.indices
            cases[key + "_coeffs"] = f.coeffs
            cases[key + "_resid"] = np.array([f.residual_fro])
            cases[key + "_pivots"] = q.pivots
            cases[key + "_r"] = q.r
            cases[key + "_q"] = q.q
    # tolerance rule on a noisy rank-4 product
    for si, tol in enumerate([0.5, 1e-2, 1e-6]):
        a = ref.matmul(port.seeded_matrix(25, 4, 60 + si), port.seeded_matrix(4, 30, 70 + si))
        a = a + 1e-7 * port.seeded_matrix(25, 30, 80 + si)
        f = ref.column_id(a, tol=tol)
        key = f"tol_{si}"
        cases[key + "_a"] = a
        cases[key + "_tol"] = np.array([tol])
        cases[key + "_indices"] = f.indices
        cases[key + "_coeffs"] = f.coeffs
        cases[key + "_resid"] = np.array([f.residual_fro])
    # sub_id with strided specs (grid.cpp:62-130, id.cpp:54-60)
    for si, (dims, strides, per) in enumerate([([24], [3], [False]), ([20, 20], [2, 2], [True, True]),
                                               ([9, 7], [2, 2], [False, False]),
                                               ([12, 10, 8], [3, 3, 3], [False] * 3)]):
        m = int(np.prod(dims))
        a = port.seeded_matrix(m, 13, 300 + si)
        f = ref.sub_id(a, dims, strides, rank=3, periodic=per)
        key = f"sub_{si}"
        cases[key + "_a_sha"] = digest(a)
        cases[key + "_seed"] = np.array([300 + si], dtype=np.int64)
        cases[key + "_dims"] = np.array(dims, dtype=np.int64)
        cases[key + "_strides"] = np.array(strides, dtype=np.int64)
        cases[key + "_periodic"] = np.array(per, dtype=np.int64)
        cases[key + "_rows"] = ref.row_indices(dims, strides, per)
        cases[key + "_indices"] = f.indices
        cases[key + "_coeffs"] = f.coeffs
        cases[key + "_resid"] = np.array([f.residual_fro])
    # Gaussian-sketch path restated through the reference's matmul + column_id
    for si, (m, n, ell, k) in enumerate([(2000, 100, 20, 10), (1500, 64, 48, 32)]):
        a = port.seeded_matrix(m, n, 900 + si)
        om = port.gaussian(ell, m, 950 + si)
        y = ref.matmul(om, a)
        f = ref.column_id(y, rank=k)
        key = f"sk_{si}"
        cases[key + "_shape"] = np.array([m, n, ell, 900 + si, 950 + si], dtype=np.int64)
        cases[key + "_a_sha"] = digest(a)
        cases[key + "_omega_sha"] = digest(om)
        cases[key + "_y"] = y
        cases[key + "_k"] = np.array([k])
        cases[key + "_indices"] = f.indices
        cases[key + "_coeffs"] = f.coeffs
        cases[key + "_resid"] = np.array([f.residual_fro])
    np.savez_compressed(os.path.join(OUT, "reference_cases.npz"), **cases)
    print("wrote", len(cases), "arrays")


if __name__ == "__main__":
    main()
