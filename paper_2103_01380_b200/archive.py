"""Archive codec surface: the reference's spid/archive.hpp API
(proj/include/spid/archive.hpp:41-76) and the CLI's batch compression of a
whole structured field (proj/tools/spid_cli.cpp:195-232), each a call into
the C ABI (include/spidgpu.h, "Archive codec").

    data = compress_field(a, dims=(64, 64, 64), blocks=(4, 4, 4), strides=(2, 2, 2), rank=8)
    approx = decompress(data)        # == reference spid::decompress(decode(data))
    info = archive_info_json(data)   # == spid::archive_info_json(decode(data))

Archives are plain `bytes` in the reference's container format (magic "SPID",
u32 version 1, JSON metadata section, CRC-32 framed block sections), so a
file written by either side is read by the other.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .spid import RankRule, SpidError, _rule

__all__ = ["compress_field", "decompress", "archive_info_json", "archive_shape", "crc32",
           "ARCHIVE_EXACT", "ARCHIVE_SKETCH"]

ARCHIVE_EXACT, ARCHIVE_SKETCH = N.ARCHIVE_EXACT, N.ARCHIVE_SKETCH


def _is_cuda(a) -> bool:
    return hasattr(a, "is_cuda") and a.is_cuda


def compress_field(a, dims, blocks=None, strides=None, rank=None, tol=None, *, periodic=None,
                   qoi="", provenance="", mode=ARCHIVE_EXACT, ell=0, seed=0, rule: RankRule | None = None,
                   out=None, device=0):
    """Batch SPID archive of a field: one spid() per block of
    make_block_domains(grid, blocks) with SubsampleSpec::strided(local,
    strides, include_boundary=True), then encode().

    `a` is m x n with rows = grid points (axis 0 fastest): a numpy array
    (copied to the device inside the call) or a CUDA torch tensor in
    column-major layout (a.T contiguous), used in place. mode=ARCHIVE_EXACT
    reproduces the reference's archive byte for byte; ARCHIVE_SKETCH puts an
    ell-row Gaussian sketch (Philox, `seed`) in front of each block's column ID.

    Returns the archive as bytes, or -- when `out` (a uint8 buffer at least as
    large as the archive) is given -- copies it there and returns its length.
    """
    nax = len(dims)
    blocks = list(blocks) if blocks is not None else [1] * nax
    strides = list(strides) if strides is not None else [1] * nax
    rr = _rule(rank, tol, rule)
    spec = N.archive_spec(dims, blocks, strides, periodic, mode, ell, seed, qoi, provenance)
    h = N.handle(device)
    nbytes = C.c_int64()
    if _is_cuda(a):
        m, n = a.shape
        lda = a.stride(1)
        if a.stride(0) != 1:
            raise ValueError("device input must be column-major (a.T contiguous)")
        rc = N.lib.spidgpu_archive_compress(h.h, C.c_void_p(a.data_ptr()), m, n, lda, 1, C.byref(spec),
                                            C.byref(rr.c()), C.byref(nbytes))
    else:
        af = np.asfortranarray(np.asarray(a, dtype=np.float64))
        if af.ndim != 2:
            raise ValueError("expected a 2-D array")
        m, n = af.shape
        rc = N.lib.spidgpu_archive_compress(h.h, C.c_void_p(af.ctypes.data), m, n, max(m, 1), 0,
                                            C.byref(spec), C.byref(rr.c()), C.byref(nbytes))
    h.check(rc)
    if out is not None:  # caller-owned buffer (numpy uint8 or pinned torch tensor)
        ptr = out.data_ptr() if hasattr(out, "data_ptr") else out.ctypes.data
        cap = out.numel() if hasattr(out, "numel") else out.size
        h.check(N.lib.spidgpu_archive_fetch(h.h, C.c_void_p(ptr), cap))
        return nbytes.value
    view, n = C.c_void_p(), C.c_int64()
    h.check(N.lib.spidgpu_archive_view(h.h, C.byref(view), C.byref(n)))
    return C.string_at(view.value, n.value) if n.value else b""


def _buf(data):
    """Zero-copy uint8 view of an archive held in bytes / bytearray / mmap /
    numpy memory (a page-locked buffer stays page-locked, so the library
    uploads it directly instead of staging it)."""
    if isinstance(data, np.ndarray):
        b = np.ascontiguousarray(data).reshape(-1).view(np.uint8)
    else:
        b = np.frombuffer(memoryview(data).cast("B"), dtype=np.uint8)
    return b, C.c_void_p(b.ctypes.data if b.size else 0)


def archive_shape(data) -> tuple[int, int, int]:
    """(rows, cols, block count) of the matrix decompress() returns."""
    b, p = _buf(data)
    rows, cols, blocks = C.c_int64(), C.c_int64(), C.c_int64()
    rc = N.lib.spidgpu_archive_shape(p, b.size, C.byref(rows), C.byref(cols), C.byref(blocks))
    if rc:
        raise SpidError(N.status_name(rc), "archive header")
    return rows.value, cols.value, blocks.value


def decompress(data, *, out=None, device=0) -> np.ndarray:
    """spid::decompress(spid::decode(data)) (proj/src/archive.cpp:214-249,
    281-303). Returns a Fortran-order float64 array, or writes into `out`
    (a CUDA torch tensor, column-major) and returns it."""
    b, p = _buf(data)
    h = N.handle(device)
    if out is not None and _is_cuda(out):
        if out.stride(0) != 1:
            raise ValueError("device output must be column-major (out.T contiguous)")
        h.check(N.lib.spidgpu_archive_decompress(h.h, p, b.size, C.c_void_p(out.data_ptr()), out.stride(1), 1))
        return out
    try:
        rows, cols, _ = archive_shape(data)
    except SpidError:
        rows = cols = 0
    res = np.empty((max(rows, 1), max(cols, 1)), dtype=np.float64, order="F")
    # a malformed archive fails inside the call with the reference's error name
    h.check(N.lib.spidgpu_archive_decompress(h.h, p, b.size, C.c_void_p(res.ctypes.data), max(rows, 1), 0))
    return res


def archive_info_json(data, *, device=0) -> str:
    """spid::archive_info_json(decode(data)) (proj/src/archive.cpp:260-268)."""
    b, p = _buf(data)
    h = N.handle(device)
    n = C.c_int64()
    h.check(N.lib.spidgpu_archive_info(h.h, p, b.size, None, 0, C.byref(n)))
    out = C.create_string_buffer(n.value + 1)
    h.check(N.lib.spidgpu_archive_info(h.h, p, b.size, out, n.value + 1, C.byref(n)))
    return out.value.decode()


def crc32(data, *, device=0) -> int:
    """spid::crc32 (proj/src/archive.cpp:168-178), computed on the device."""
    h = N.handle(device)
    v = C.c_uint32()
    if _is_cuda(data):
        h.check(N.lib.spidgpu_crc32(h.h, C.c_void_p(data.data_ptr()), data.numel() * data.element_size(), 1,
                                    C.byref(v)))
    else:
        b, p = _buf(data)
        h.check(N.lib.spidgpu_crc32(h.h, p, b.size, 0, C.byref(v)))
    return v.value
