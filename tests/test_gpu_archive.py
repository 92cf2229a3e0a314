"""GPU parity of the archive codec through the C ABI:

* spidgpu_crc32 == CRC-32/ISO-HDLC (reference vector, zlib, the port);
* spidgpu_archive_compress(EXACT) == the reference CLI's batch archive, byte
  for byte (tests/golden/archive_cases.npz, written by oracle/_ref);
* spidgpu_archive_decompress == the reference's decompress, bit for bit;
* spidgpu_archive_info == archive_info_json;
* the reference's error names for corrupt archives and bad plans;
* SKETCH-mode archives decode and decompress identically on both sides.
"""
import hashlib
import json
import os
import zlib

import numpy as np
import pytest
import torch

from oracle import archive_port as AP

pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "archive_cases.npz"))
NCASES = len([k for k in GOLD.files if k.endswith("_bytes")])


@pytest.fixture(scope="module")
def A():
    from paper_2103_01380_b200 import archive
    return archive


def _sha(a):
    return np.frombuffer(hashlib.sha256(np.asfortranarray(a).tobytes(order="F")).digest(), dtype=np.uint8)


def _case(ci):
    p = GOLD[f"arc_{ci}_params"]
    nax = int(p[0])
    dims = list(map(int, p[1:1 + nax]))
    blocks = list(map(int, p[1 + nax:1 + 2 * nax]))
    strides = list(map(int, p[1 + 2 * nax:1 + 3 * nax]))
    per = list(map(int, p[1 + 3 * nax:1 + 4 * nax]))
    rank, n = int(p[1 + 4 * nax]), int(p[2 + 4 * nax])
    tol = float(GOLD[f"arc_{ci}_tol"][0])
    kw = dict(rank=rank) if rank > 0 else dict(tol=tol)
    return GOLD[f"arc_{ci}_a"], dims, blocks, strides, per, kw


def test_crc32_reference_vector(A):
    assert A.crc32(b"123456789") == 0xCBF43926
    assert A.crc32(b"") == 0


@pytest.mark.parametrize("n", [1, 7, 8, 1023, 1024, 1025, 262144 + 5, 3 << 20])
def test_crc32_matches_zlib(A, n):
    data = np.random.default_rng(n).integers(0, 256, n, dtype=np.uint8).tobytes()
    assert A.crc32(data) == zlib.crc32(data)


@pytest.mark.parametrize("n", [(8 << 20) + 3, (37 << 20) + 11])
def test_crc32_staged_upload(A, n):
    """Pageable host buffers >= 8 MB go through the threaded pinned staging
    (4 MB chunks, ragged tail); a page-locked buffer of the same bytes is
    copied directly. Both equal zlib."""
    data = np.random.default_rng(n).integers(0, 256, n, dtype=np.uint8)
    want = zlib.crc32(data.tobytes())
    assert A.crc32(data.tobytes()) == want
    pinned = torch.from_numpy(data).pin_memory()
    assert A.crc32(pinned.numpy()) == want
    assert A.crc32(data.tobytes()) == want  # staging slots reused across calls


@pytest.mark.parametrize("off", [0, 1, 3, 8, 13])
def test_crc32_device_unaligned(A, off):
    buf = torch.randint(0, 256, (70001,), dtype=torch.uint8, device="cuda")
    view = buf[off:off + 65537]
    assert A.crc32(view) == zlib.crc32(view.cpu().numpy().tobytes())


@pytest.mark.parametrize("ci", range(NCASES))
def test_compress_field_bytes_identical(A, ci):
    a, dims, blocks, strides, per, kw = _case(ci)
    data = A.compress_field(a, dims, blocks, strides, periodic=per, qoi=f"q{ci}",
                            provenance="golden fixture", **kw)
    ref = GOLD[f"arc_{ci}_bytes"].tobytes()
    assert len(data) == len(ref)
    assert data == ref


@pytest.mark.parametrize("ci", range(NCASES))
def test_compress_field_device_input(A, ci):
    a, dims, blocks, strides, per, kw = _case(ci)
    at = torch.from_numpy(np.ascontiguousarray(a.T)).cuda().T  # column-major view
    data = A.compress_field(at, dims, blocks, strides, periodic=per, qoi=f"q{ci}",
                            provenance="golden fixture", **kw)
    assert data == GOLD[f"arc_{ci}_bytes"].tobytes()


@pytest.mark.parametrize("ci", range(NCASES))
def test_decompress_bit_identical(A, ci):
    data = GOLD[f"arc_{ci}_bytes"].tobytes()
    out = A.decompress(data)
    assert np.array_equal(_sha(out), GOLD[f"arc_{ci}_out_sha"])
    rows, cols, nblk = A.archive_shape(data)
    assert out.shape == (rows, cols)


@pytest.mark.parametrize("ci", [0, 1, 5])
def test_decompress_to_device(A, ci):
    data = GOLD[f"arc_{ci}_bytes"].tobytes()
    rows, cols, _ = A.archive_shape(data)
    out = torch.empty((cols, rows + 3), dtype=torch.float64, device="cuda").T  # ld = rows + 3
    A.decompress(data, out=out)
    host = np.asfortranarray(out[:rows].cpu().numpy())
    assert np.array_equal(_sha(host), GOLD[f"arc_{ci}_out_sha"])


@pytest.mark.parametrize("ci", range(NCASES))
def test_archive_info_identical(A, ci):
    data = GOLD[f"arc_{ci}_bytes"].tobytes()
    assert A.archive_info_json(data) == GOLD[f"arc_{ci}_info"].tobytes().decode()


def test_archive_rejects_corruption(A):
    data = bytearray(GOLD["arc_0_bytes"].tobytes())
    cases = []
    c = bytearray(data)
    c[len(c) // 2] ^= 0x40
    cases.append(("ChecksumMismatch", c))
    c = bytearray(data)
    c[4] += 1
    cases.append(("VersionUnsupported", c))
    c = bytearray(data)
    c[0] = ord("X")
    cases.append(("BadMagic", c))
    cases.append(("TruncatedPayload", data[:-7]))
    c = bytearray(data)
    c[20] ^= 0x01  # inside the metadata JSON
    cases.append(("ChecksumMismatch", c))
    cases.append(("TruncatedPayload", data + b"\0"))
    for name, bad in cases:
        with pytest.raises(Exception) as e:
            A.decompress(bytes(bad))
        assert getattr(e.value, "name", None) == name, (name, e.value)
        with pytest.raises(AP.ArchiveError) as e2:
            AP.decode(bytes(bad))
        assert e2.value.name == name


def test_compress_field_errors(A):
    rng = np.random.default_rng(3)
    a = rng.standard_normal((10 * 10, 6))
    cases = [
        ("BlockTooSmall", dict(dims=(10, 10), blocks=(11, 1), strides=(2, 2), rank=2)),
        ("BlockTooSmall", dict(dims=(10, 10), blocks=(0, 1), strides=(2, 2), rank=2)),
        ("BadGridGeom", dict(dims=(1, 100), blocks=(1, 1), strides=(1, 1), rank=2)),
        ("BadRankRule", dict(dims=(10, 10), blocks=(2, 2), strides=(2, 2), tol=1.5)),
        ("BadSubsampleSpec", dict(dims=(10, 10), blocks=(2, 2), strides=(0, 2), rank=2)),
        ("RankUnreachable", dict(dims=(10, 10), blocks=(2, 2), strides=(2, 2), rank=7)),
    ]
    for name, kw in cases:
        dims, blocks, strides = kw.pop("dims"), kw.pop("blocks"), kw.pop("strides")
        with pytest.raises(Exception) as e:
            A.compress_field(a, dims, blocks, strides, **kw)
        assert getattr(e.value, "name", None) == name, (name, e.value)
    with pytest.raises(Exception) as e:  # select_rows past the matrix
        A.compress_field(a[:90], (10, 10), (2, 2), (2, 2), rank=2)
    assert e.value.name == "IndexOutOfRange"
    bad = a.copy()
    bad[11, 3] = np.nan  # a FINE row (not on the coarse grid) of block 0
    with pytest.raises(Exception) as e:
        A.compress_field(bad, (10, 10), (2, 2), (2, 2), rank=2)
    assert e.value.name == "NonFiniteInput"


def test_compress_field_zero_block(A):
    a = np.random.default_rng(4).standard_normal((12 * 12, 5))
    a[:6, :] = 0.0  # not a whole block -> fine
    A.compress_field(a, (12, 12), (2, 2), (2, 2), rank=1)
    z = a.copy()
    blk = AP.make_block_domains([12, 12], [0, 0], [2, 2])[1][0]
    z[blk, :] = 0.0
    with pytest.raises(Exception) as e:
        A.compress_field(z, (12, 12), (2, 2), (2, 2), rank=1)
    assert e.value.name == "ZeroMatrix"


def test_sketch_archive_roundtrip(A, ref):
    """SKETCH mode: a valid archive the reference decodes; both sides'
    decompress agree bitwise; the error stays close to the exact archive's."""
    a, dims, blocks, strides, per, _ = _case(5)
    exact = A.compress_field(a, dims, blocks, strides, periodic=per, rank=5)
    sk = A.compress_field(a, dims, blocks, strides, periodic=per, rank=5, mode=A.ARCHIVE_SKETCH,
                          ell=5 + 8, seed=11)
    ours = A.decompress(sk)
    assert np.array_equal(ours, ref.archive_decompress(sk))
    info = json.loads(A.archive_info_json(sk))
    assert info["block_ranks"] == [5] * 8
    e_exact = np.linalg.norm(A.decompress(exact) - a) / np.linalg.norm(a)
    e_sk = np.linalg.norm(ours - a) / np.linalg.norm(a)
    assert e_sk < 3 * e_exact + 1e-12


def test_large_field_exact_vs_reference(A, ref):
    """64^3 grid, 64 blocks: byte-identical archive and bit-identical decompress."""
    dims, blocks, strides = (64, 64, 64), (4, 4, 4), (2, 2, 2)
    rng = np.random.default_rng(9)
    x = np.linspace(0, 2 * np.pi, 64, endpoint=False)
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    t = np.linspace(0, 1, 24)
    a = (np.outer((np.sin(X) * np.cos(Y) * np.cos(Z)).ravel(order="F"), np.exp(-t)) +
         0.3 * np.outer((np.cos(2 * X) * np.sin(Y + Z)).ravel(order="F"), np.cos(3 * t)) +
         1e-5 * rng.standard_normal((64 ** 3, 24)))
    a = np.asfortranarray(a)
    ours = A.compress_field(a, dims, blocks, strides, periodic=(1, 1, 1), tol=1e-4, qoi="u")
    theirs = ref.compress_field(a, dims, blocks, strides, tol=1e-4, periodic=(1, 1, 1), qoi="u")
    assert ours == theirs
    assert np.array_equal(A.decompress(ours), ref.archive_decompress(theirs))


def test_large_field_property_roundtrip(A):
    """128^3 x 32 on the device only: framing decodes on the port, every CRC
    equals zlib's, decompress of the archive reproduces the coarse rows."""
    n = 32
    at = torch.randn(n, 128 ** 3, dtype=torch.float64, device="cuda").T
    data = A.compress_field(at, (128, 128, 128), (4, 4, 4), (2, 2, 2), rank=8, mode=A.ARCHIVE_SKETCH,
                            ell=16, seed=1)
    ar = AP.decode(data)  # validates every section CRC with the port
    assert len(ar.blocks) == 64
    assert AP.encode(ar) == data
    out = torch.empty((n, 128 ** 3), dtype=torch.float64, device="cuda").T
    A.decompress(data, out=out)
    assert torch.isfinite(out).all()
    # the archive (> 8 MB) from pageable bytes went through the staged upload;
    # from page-locked memory it is copied directly: same result bit for bit
    assert len(data) > (8 << 20)
    pinned = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
    out2 = torch.empty_like(out.T).T
    A.decompress(pinned.numpy(), out=out2)
    assert torch.equal(out, out2)
