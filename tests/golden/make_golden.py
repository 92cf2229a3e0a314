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
    archive_cases(ref, port)


def smooth_field(dims, n, seed):
    """Deterministic smooth snapshots on a structured grid (rows = points,
    axis 0 fastest): a few separable Fourier modes with decaying amplitudes,
    each with its own temporal frequency, plus a little seeded noise."""
    rng = np.random.default_rng(seed)
    axes = np.meshgrid(*[np.arange(d) / d for d in dims], indexing="ij")
    t = np.linspace(0.0, 1.0, n)
    a = np.zeros((int(np.prod(dims)), n))
    for mode in range(6):
        ks = rng.integers(1, 3, size=len(dims))
        ph = rng.uniform(0, 2 * np.pi, size=len(dims))
        shape = np.ones_like(axes[0])
        for ax, k, p in zip(axes, ks, ph):
            shape = shape * np.sin(2 * np.pi * k * ax + p)
        a += (0.5 ** mode) * np.outer(shape.ravel(order="F"), np.cos(2 * np.pi * (mode + 1) * t + mode))
    return np.asfortranarray(a + 1e-6 * rng.standard_normal(a.shape))


# (dims, blocks, strides, periodic, rank, tol, snapshots, input kind)
ARCHIVE_CASES = [
    ((10, 10), (2, 2), (2, 2), (1, 1), 1, 0.0, 20, "smooth"),
    ((13, 11, 9), (3, 2, 2), (2, 3, 1), (0, 1, 0), 0, 1e-3, 15, "smooth"),
    ((17,), (3,), (4,), (0,), 2, 0.0, 9, "seeded"),
    ((12, 8), (1, 1), (1, 1), (1, 1), 4, 0.0, 10, "seeded"),
    ((9, 7, 6), (9, 1, 2), (2, 2, 2), (0, 0, 0), 1, 0.0, 6, "seeded"),
    ((12, 12, 12), (2, 2, 2), (2, 2, 2), (1, 1, 1), 5, 0.0, 16, "smooth"),
    ((20, 14), (3, 2), (3, 2), (0, 0), 0, 1e-6, 12, "smooth"),
]


def archive_cases(ref, port):
    """Archives of the CLI's batch compression (spid_cli.cpp:195-232 +
    archive.cpp encode) and their decompress(), from the reference."""
    cases = {}
    for ci, (dims, blocks, strides, per, rank, tol, n, kind) in enumerate(ARCHIVE_CASES):
        m = int(np.prod(dims))
        a = smooth_field(dims, n, 77 + ci) if kind == "smooth" else port.seeded_matrix(m, n, 500 + ci)
        data = ref.compress_field(a, dims, blocks, strides, rank=rank, tol=tol, periodic=per,
                                  qoi=f"q{ci}", provenance="golden fixture")
        out = ref.archive_decompress(data)
        key = f"arc_{ci}"
        cases[key + "_a"] = a
        cases[key + "_params"] = np.array([len(dims), *dims, *blocks, *strides, *per, rank, n], dtype=np.int64)
        cases[key + "_tol"] = np.array([tol])
        cases[key + "_bytes"] = np.frombuffer(data, dtype=np.uint8).copy()
        cases[key + "_out_sha"] = digest(out)
        cases[key + "_info"] = np.frombuffer(ref.archive_info(data).encode(), dtype=np.uint8).copy()
    cases["crc_kat"] = np.array([ref.crc32(b"123456789")], dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "archive_cases.npz"), **cases)
    print("wrote", len(cases), "archive arrays")
    pipeline_cases(ref, port)


# (dims, blocks, strides, periodic, include_boundary, time_chunk, stage1_rank,
#  stage2_tol, snapshots, input kind)
PIPELINE_CASES = [
    ((10, 10), (2, 2), (2, 2), (1, 1), True, 8, 1, 1e-6, 20, "smooth"),
    ((12, 10), (2, 2), (2, 2), (1, 0), True, 5, 2, 1e-8, 23, "lowrank"),
    ((13, 11, 9), (3, 2, 2), (2, 3, 1), (0, 1, 0), True, 4, 3, 1e-6, 14, "smooth"),
    ((17,), (3,), (4,), (0,), True, 3, 2, 1e-10, 10, "lowrank"),
    ((14,), (1,), (1,), (0,), True, 9, 5, 1e-6, 9, "lowrank"),       # batch-equivalent single chunk
    ((9, 7, 6), (9, 1, 2), (2, 2, 2), (0, 0, 0), True, 2, 1, 1e-6, 7, "seeded"),
    ((12, 12, 12), (2, 2, 2), (2, 2, 2), (1, 1, 1), True, 6, 4, 1e-7, 16, "smooth"),
    ((16, 12), (2, 3), (3, 2), (0, 0), False, 7, 3, 1e-6, 15, "smooth"),  # no boundary pinning
]


def pipeline_cases(ref, port):
    """Archives of run_pipeline (proj/src/pipeline.cpp:104-294) + encode()."""
    rng = np.random.default_rng(2024)
    cases = {}
    for ci, (dims, blocks, strides, per, incl, T, k, tol, n, kind) in enumerate(PIPELINE_CASES):
        m = int(np.prod(dims))
        if kind == "smooth":
            a = smooth_field(dims, n, 300 + ci)
        elif kind == "lowrank":
            a = np.asfortranarray(rng.standard_normal((m, 3)) @ rng.standard_normal((3, n)) +
                                  1e-4 * rng.standard_normal((m, n)))
        else:
            a = port.seeded_matrix(m, n, 700 + ci)
        data, stats = ref.run_pipeline(a, dims, blocks, strides, T, k, tol, periodic=per,
                                       include_boundary=incl, qoi=f"p{ci}", provenance="golden pipeline")
        key = f"pipe_{ci}"
        cases[key + "_a"] = a
        cases[key + "_params"] = np.array([len(dims), *dims, *blocks, *strides, *per, int(incl), T, k, n],
                                          dtype=np.int64)
        cases[key + "_tol"] = np.array([tol])
        cases[key + "_bytes"] = np.frombuffer(data, dtype=np.uint8).copy()
        cases[key + "_stats"] = np.array(stats, dtype=np.int64)
        try:
            cases[key + "_out_sha"] = digest(ref.archive_decompress(data))
        except oracle.OracleError as e:  # e.g. ExtrapolationRequired without boundary pinning
            cases[key + "_out_err"] = np.frombuffer(e.name.encode(), dtype=np.uint8).copy()
    np.savez_compressed(os.path.join(OUT, "pipeline_cases.npz"), **cases)
    print("wrote", len(cases), "pipeline arrays")


if __name__ == "__main__":
    main()
