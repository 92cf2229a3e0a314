"""TEST INFRASTRUCTURE ONLY -- a Python restatement of the reference archive
container (proj/src/archive.cpp) used as a checker, never by the product.

    crc32(data)                  archive.cpp:168-178 (bitwise CRC-32/ISO-HDLC)
    encode(meta, blocks)         archive.cpp:193-212 (+ put_section :83-88,
                                 put_index_array :100-103, put_matrix :110-116)
    decode(data)                 archive.cpp:214-249 (same error names/order)
    meta_json(meta)              meta_to_json(...).dump(), archive.cpp:119-136
    decompress(archive, port)    archive.cpp:281-303 via the C oracle's
                                 interp_apply and matmul (bit-exact restatements)
    make_block_domains(...)      blocking.cpp:12-104
"""
from __future__ import annotations

import json
import struct
from dataclasses import dataclass, field

import numpy as np

_POLY = 0xEDB88320
_TABLE = []
for _i in range(256):
    _c = _i
    for _ in range(8):
        _c = (_c >> 1) ^ (_POLY & -(_c & 1))
    _TABLE.append(_c & 0xFFFFFFFF)


class ArchiveError(RuntimeError):
    def __init__(self, name: str):
        super().__init__(name)
        self.name = name


def crc32_bitwise(data: bytes) -> int:
    """The reference loop, bit by bit (small inputs only)."""
    crc = 0xFFFFFFFF
    for byte in data:
        crc ^= byte
        for _ in range(8):
            crc = (crc >> 1) ^ (_POLY & (-(crc & 1) & 0xFFFFFFFF))
    return (~crc) & 0xFFFFFFFF


def crc32(data: bytes) -> int:
    """Same function, bytewise table form (identical results, faster); large
    inputs go through zlib.crc32, the same CRC-32/ISO-HDLC (cross-checked in
    tests/test_archive_oracle.py)."""
    if len(data) > 4096:
        import zlib
        return zlib.crc32(data) & 0xFFFFFFFF
    crc = 0xFFFFFFFF
    for byte in data:
        crc = _TABLE[(crc ^ byte) & 0xFF] ^ (crc >> 8)
    return (~crc) & 0xFFFFFFFF


@dataclass
class Block:
    coarse: bool
    union_indices: list
    skeleton_indices: list
    skeleton: np.ndarray  # Fortran float64
    coeffs: np.ndarray


@dataclass
class Archive:
    meta: dict
    blocks: list = field(default_factory=list)


def meta_json(meta: dict) -> bytes:
    """nlohmann's dump(): keys sorted, no whitespace. Floats are written with
    repr(), which matches nlohmann's shortest round-trip form for the values
    the metadata carries (tolerances in (0, 1) and 0.0)."""
    return json.dumps(meta, sort_keys=True, separators=(",", ":"), ensure_ascii=False).encode()


def _section(payload: bytes) -> bytes:
    return struct.pack("<Q", len(payload)) + payload + struct.pack("<I", crc32(payload))


def _index_array(idx) -> bytes:
    return struct.pack("<Q", len(idx)) + np.asarray(idx, dtype="<u8").tobytes()


def _matrix(m: np.ndarray) -> bytes:
    m = np.asfortranarray(m, dtype=np.float64)
    return struct.pack("<QQ", m.shape[0], m.shape[1]) + m.tobytes(order="F")


def encode(ar: Archive) -> bytes:
    out = [b"SPID", struct.pack("<I", 1), _section(meta_json(ar.meta)), struct.pack("<Q", len(ar.blocks))]
    for b in ar.blocks:
        payload = (bytes([1 if b.coarse else 0]) + _index_array(b.union_indices) +
                   _index_array(b.skeleton_indices) + _matrix(b.skeleton) + _matrix(b.coeffs))
        out.append(_section(payload))
    return b"".join(out)


class _Reader:
    def __init__(self, data: bytes):
        self.d, self.at = data, 0

    def take(self, n: int) -> bytes:
        if self.at + n > len(self.d):
            raise ArchiveError("TruncatedPayload")
        v = self.d[self.at:self.at + n]
        self.at += n
        return v

    def u32(self) -> int:
        return struct.unpack("<I", self.take(4))[0]

    def u64(self) -> int:
        return struct.unpack("<Q", self.take(8))[0]

    def section(self) -> bytes:
        payload = self.take(self.u64())
        if self.u32() != crc32(payload):
            raise ArchiveError("ChecksumMismatch")
        return payload


def decode(data: bytes) -> Archive:
    r = _Reader(data)
    if r.take(4) != b"SPID":
        raise ArchiveError("BadMagic")
    if r.u32() != 1:
        raise ArchiveError("VersionUnsupported")
    try:
        meta = json.loads(r.section().decode())
    except (ValueError, UnicodeDecodeError):
        raise ArchiveError("TruncatedPayload")
    ar = Archive(meta)
    for _ in range(r.u64()):
        br = _Reader(r.section())
        coarse = br.take(1)[0] != 0
        arrays = []
        for _a in range(2):
            cnt = br.u64()
            arrays.append(list(np.frombuffer(br.take(8 * cnt), dtype="<u8").astype(np.int64)))
        mats = []
        for _m in range(2):
            rows, cols = br.u64(), br.u64()
            if rows == 0 or cols == 0:
                raise ArchiveError("TruncatedPayload")
            mats.append(np.frombuffer(br.take(8 * rows * cols), dtype="<f8").reshape(cols, rows).T.copy(order="F"))
        if br.at != len(br.d):
            raise ArchiveError("TruncatedPayload")
        ar.blocks.append(Block(coarse, arrays[0], arrays[1], mats[0], mats[1]))
    if r.at != len(data):
        raise ArchiveError("TruncatedPayload")
    return ar


def _axis_segments(dim, count):
    if count < 1 or count > dim:
        raise ArchiveError("BlockTooSmall")
    base, at, segs = dim // count, 0, []
    for b in range(count):
        ln = dim - at if b + 1 == count else base
        segs.append((at, ln))
        at += ln
    return segs


def make_block_domains(dims, periodic, blocks):
    """[(rows (global, local order), local dims, local periodic)] in block order."""
    nax = len(dims)
    segs = [_axis_segments(dims[a], blocks[a]) for a in range(nax)] + [[(0, 1)]] * (3 - nax)
    d0 = dims[0]
    d1 = dims[1] if nax > 1 else 1
    out = []
    for s2, l2 in segs[2]:
        for s1, l1 in segs[1]:
            for s0, l0 in segs[0]:
                i0, i1, i2 = np.meshgrid(np.arange(l0), np.arange(l1), np.arange(l2), indexing="ij")
                rows = ((s0 + i0) + d0 * (s1 + i1) + d0 * d1 * (s2 + i2)).ravel(order="F")
                ld = [l0, l1, l2][:nax]
                lp = [bool(periodic[a]) and ld[a] == dims[a] for a in range(nax)]
                out.append((rows, ld, lp))
    return out


def decompress(ar: Archive, port) -> np.ndarray:
    """archive.cpp:281-303 with the C oracle's bit-exact interp_apply/matmul."""
    g = ar.meta["grid"]
    doms = make_block_domains(g["dims"], g["periodic"], ar.meta["blocks_per_axis"])
    if len(doms) != len(ar.blocks):
        raise ArchiveError("CoverageGap")
    total = sum(len(r) for r, _, _ in doms)
    out = np.zeros((total, ar.blocks[0].coeffs.shape[1]), order="F")
    for (rows, ld, lp), b in zip(doms, ar.blocks):
        skel = b.skeleton
        if b.coarse:
            skel = port.interp_apply(ld, ar.meta["strides"], skel, lp, ar.meta["include_boundary"])
        out[rows, :] = port.matmul(skel, b.coeffs)
    return out
