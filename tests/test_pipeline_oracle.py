"""CPU: the streaming two-stage restatement (oracle/pipeline_port.py over the
C oracle) pinned against the reference's own run_pipeline archives
(tests/golden/pipeline_cases.npz, written by oracle/_ref)."""
import hashlib
import os

import numpy as np
import pytest

import oracle
from oracle import archive_port as AP
from oracle import pipeline_port as PP

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "pipeline_cases.npz"))
NCASES = len([k for k in GOLD.files if k.endswith("_bytes")])


def case(ci):
    p = GOLD[f"pipe_{ci}_params"]
    nax = int(p[0])
    dims = list(map(int, p[1:1 + nax]))
    blocks = list(map(int, p[1 + nax:1 + 2 * nax]))
    strides = list(map(int, p[1 + 2 * nax:1 + 3 * nax]))
    per = list(map(int, p[1 + 3 * nax:1 + 4 * nax]))
    incl, T, k, n = (int(x) for x in p[1 + 4 * nax:5 + 4 * nax])
    return dict(a=GOLD[f"pipe_{ci}_a"], dims=dims, blocks=blocks, strides=strides, periodic=per,
                include_boundary=bool(incl), time_chunk=T, stage1_rank=k,
                stage2_tol=float(GOLD[f"pipe_{ci}_tol"][0]), n=n)


@pytest.mark.parametrize("ci", range(NCASES))
def test_port_reproduces_reference_pipeline(ci):
    c = case(ci)
    ar = PP.run_pipeline(c["a"], c["dims"], c["blocks"], c["strides"], c["time_chunk"], c["stage1_rank"],
                         c["stage2_tol"], oracle.port(), periodic=c["periodic"],
                         include_boundary=c["include_boundary"], qoi=f"p{ci}", provenance="golden pipeline")
    assert AP.encode(ar) == GOLD[f"pipe_{ci}_bytes"].tobytes()


@pytest.mark.parametrize("ci", range(NCASES))
def test_pipeline_archive_structure(ci):
    c = case(ci)
    ar = AP.decode(GOLD[f"pipe_{ci}_bytes"].tobytes())
    assert ar.meta["mode"] == "two-stage" and ar.meta["time_chunk"] == c["time_chunk"]
    nchunks = -(-c["n"] // c["time_chunk"])
    stats = GOLD[f"pipe_{ci}_stats"]
    assert stats[2] == nchunks * len(ar.blocks) and stats[3] == len(ar.blocks)
    for b in ar.blocks:
        assert b.union_indices == sorted(b.union_indices)
        assert set(b.skeleton_indices) <= set(b.union_indices)
        assert b.coeffs.shape == (len(b.skeleton_indices), c["n"])
        assert len(b.union_indices) <= nchunks * c["stage1_rank"]


@pytest.mark.parametrize("ci", range(NCASES))
def test_pipeline_decompress_port(ci):
    ar = AP.decode(GOLD[f"pipe_{ci}_bytes"].tobytes())
    if f"pipe_{ci}_out_err" in GOLD.files:
        with pytest.raises(Exception):
            AP.decompress(ar, oracle.port())
        return
    out = AP.decompress(ar, oracle.port())
    sha = np.frombuffer(hashlib.sha256(np.asfortranarray(out).tobytes(order="F")).digest(), dtype=np.uint8)
    assert np.array_equal(sha, GOLD[f"pipe_{ci}_out_sha"])
