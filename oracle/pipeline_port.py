"""TEST INFRASTRUCTURE ONLY -- restatement of the reference's streaming
two-stage compressor used as a checker:

    run_pipeline(a, ...)       proj/src/pipeline.cpp:104-294 (serial order)
    stage1 (per chunk)         stage1_compress_coarse, blocking.cpp:112-115
                               -> the C oracle's column_id_at_most
    stage2_compress            blocking.cpp:128-204: sorted union, concat,
                               column_id(tolerance), composed C1 * C0'
                               (same loop order, one rounding per operation)

Builds an archive_port.Archive whose encode() must equal the reference's bytes.
"""
from __future__ import annotations

import numpy as np

from . import archive_port as AP


def _stage2(stage1, chunk_starts, tol, port):
    """stage2_compress (blocking.cpp:128-204) on [(indices, coeffs, skeleton)]."""
    entries = []
    for j, (idx, _c, _s) in enumerate(stage1):
        for l, i in enumerate(idx):
            entries.append((chunk_starts[j] + int(i), j, l))
    entries.sort(key=lambda e: e[0])
    union = [e[0] for e in entries]
    m_s = stage1[0][2].shape[0]
    concat = np.zeros((m_s, len(entries)), order="F")
    for u, (_g, j, l) in enumerate(entries):
        concat[:, u] = stage1[j][2][:, l]
    second = port.column_id(concat, tol=tol)
    n_total = chunk_starts[-1] + stage1[-1][1].shape[1]
    k2 = second.rank
    final = np.zeros((k2, n_total), order="F")
    C1 = second.coeffs
    for u, (_g, j, l) in enumerate(entries):  # blocking.cpp:187-200, same order
        c0row = stage1[j][1][l]
        col0 = chunk_starts[j]
        for t in range(c0row.shape[0]):
            c0 = c0row[t]
            if c0 == 0.0:
                continue
            final[:, col0 + t] = final[:, col0 + t] + C1[:, u] * c0  # rounded mul, rounded add
    if not np.all(np.isfinite(final)):
        raise AP.ArchiveError("NonFiniteCoeffs")
    final_global = [union[p] for p in second.indices]
    return union, final_global, concat[:, second.indices], final


def run_pipeline(a, dims, blocks, strides, time_chunk, stage1_rank, stage2_tol, port,
                 periodic=None, include_boundary=True, qoi="", provenance=""):
    nax = len(dims)
    periodic = list(periodic) if periodic else [0] * nax
    m, n = a.shape
    if n == 0:
        raise AP.ArchiveError("ShortStream")
    doms = AP.make_block_domains(list(dims), periodic, list(blocks))
    blocks_out = []
    for rows, ld, lp in doms:
        J = port.row_indices(ld, list(strides), lp, include_boundary)
        coarse_rows = rows[J]
        stage1, starts = [], []
        for c0 in range(0, n, time_chunk):
            chunk = np.asfortranarray(a[coarse_rows, c0:c0 + time_chunk])
            cols = chunk.shape[1]
            f = port.column_id(chunk, rank=min(stage1_rank, cols), at_most=True)
            stage1.append((f.indices, f.coeffs, np.asfortranarray(chunk[:, f.indices])))
            starts.append(c0)
        union, fglob, fskel, fcoef = _stage2(stage1, starts, stage2_tol, port)
        blocks_out.append(AP.Block(len(J) < len(rows), union, fglob, fskel, fcoef))
    meta = {
        "grid": {"kind": "structured", "dims": list(dims), "periodic": [bool(x) for x in periodic]},
        "blocks_per_axis": list(blocks), "time_chunk": time_chunk, "strides": list(strides),
        "include_boundary": bool(include_boundary), "mode": "two-stage",
        "rank_rule": {"mode": "fixed", "k": stage1_rank, "tol": 0.0}, "stage2_tol": stage2_tol,
        "interp": "strided-multilinear", "qoi": qoi, "m": m, "n": n, "provenance": provenance,
    }
    return AP.Archive(meta, blocks_out)
