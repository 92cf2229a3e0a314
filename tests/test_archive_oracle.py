"""CPU: the archive-container port (oracle/archive_port.py) pinned against the
reference's own archives (tests/golden/archive_cases.npz, written by
oracle/_ref from the reference sources) and the reference's archive tests
(proj/tests/test_archive_metrics.cpp:61-105)."""
import hashlib
import os
import zlib

import numpy as np
import pytest

import oracle
from oracle import archive_port as AP

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "archive_cases.npz"))
NCASES = len([k for k in GOLD.files if k.endswith("_bytes")])


def _sha(a):
    return np.frombuffer(hashlib.sha256(np.asfortranarray(a).tobytes(order="F")).digest(), dtype=np.uint8)


def test_crc32_reference_vector():
    # test_archive_metrics.cpp:61-64
    assert AP.crc32_bitwise(b"123456789") == 0xCBF43926
    assert AP.crc32(b"123456789") == 0xCBF43926
    assert int(GOLD["crc_kat"][0]) == 0xCBF43926


@pytest.mark.parametrize("n", [0, 1, 7, 8, 9, 255, 1000])
def test_crc32_forms_agree(n):
    data = np.random.default_rng(n).integers(0, 256, n, dtype=np.uint8).tobytes()
    assert AP.crc32_bitwise(data) == AP.crc32(data) == zlib.crc32(data)


@pytest.mark.parametrize("ci", range(NCASES))
def test_golden_archive_roundtrip(ci):
    """decode -> encode is bitwise (test_archive_metrics.cpp:66-79) and the
    metadata section is nlohmann's compact dump of the decoded fields."""
    data = GOLD[f"arc_{ci}_bytes"].tobytes()
    ar = AP.decode(data)
    assert AP.encode(ar) == data
    mlen = int.from_bytes(data[8:16], "little")
    assert AP.meta_json(ar.meta) == data[16:16 + mlen]
    p = GOLD[f"arc_{ci}_params"]
    nax = int(p[0])
    assert ar.meta["grid"]["dims"] == list(map(int, p[1:1 + nax]))
    assert ar.meta["mode"] == "batch" and ar.meta["interp"] == "strided-multilinear"
    for b in ar.blocks:
        assert b.union_indices == sorted(b.skeleton_indices)
        assert b.coeffs.shape[0] == b.skeleton.shape[1] == len(b.skeleton_indices)


@pytest.mark.parametrize("ci", range(NCASES))
def test_golden_archive_decompress(ci):
    """The port's decompress (C-oracle interp + matmul) reproduces the
    reference's decompress bit for bit."""
    ar = AP.decode(GOLD[f"arc_{ci}_bytes"].tobytes())
    out = AP.decompress(ar, oracle.port())
    assert np.array_equal(_sha(out), GOLD[f"arc_{ci}_out_sha"])


def test_archive_rejects_corruption():
    """test_archive_metrics.cpp:81-105 on a reference archive."""
    data = bytearray(GOLD["arc_0_bytes"].tobytes())
    cases = {}
    c = bytearray(data)
    c[len(c) // 2] ^= 0x40
    cases["ChecksumMismatch"] = c
    c = bytearray(data)
    c[4] += 1
    cases["VersionUnsupported"] = c
    c = bytearray(data)
    c[0] = ord("X")
    cases["BadMagic"] = c
    cases["TruncatedPayload"] = data[:-7]
    for name, bad in cases.items():
        with pytest.raises(AP.ArchiveError) as e:
            AP.decode(bytes(bad))
        assert e.value.name == name


def test_block_domains_match_reference_plan():
    """make_block_domains: remainders go to the last block, axis 0 fastest,
    rows tile the grid exactly (blocking.cpp:12-104, 219-241)."""
    doms = AP.make_block_domains([13, 11, 9], [0, 1, 0], [3, 2, 2])
    assert len(doms) == 12
    rows = np.concatenate([r for r, _, _ in doms])
    assert np.array_equal(np.sort(rows), np.arange(13 * 11 * 9))
    assert doms[0][1] == [4, 5, 4] and doms[-1][1] == [5, 6, 5]
    assert doms[0][2] == [False, False, False]
    full = AP.make_block_domains([10, 10], [1, 1], [1, 2])
    assert full[0][2] == [True, False]  # periodic only where the block spans the axis
    with pytest.raises(AP.ArchiveError):
        AP.make_block_domains([4], [0], [5])
