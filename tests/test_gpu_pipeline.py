"""GPU parity of the streaming two-stage compressor through the
C ABI (spidgpu_stream_*): archives byte-identical to the reference's
encode(run_pipeline(...).archive) (tests/golden/pipeline_cases.npz) whatever
the push granularity, decompress bit-identical, and the reference pipeline's
error names (proj/tests/test_pipeline.cpp)."""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

from oracle import archive_port as AP

pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "pipeline_cases.npz"))
NCASES = len([k for k in GOLD.files if k.endswith("_bytes")])


def _case(ci):
    from test_pipeline_oracle import case
    return case(ci)


@pytest.fixture(scope="module")
def PL():
    from paper_2103_01380_b200 import pipeline
    return pipeline


def _cfg(PL, c, ci):
    return PL.StreamConfig(dims=c["dims"], blocks=c["blocks"], strides=c["strides"], time_chunk=c["time_chunk"],
                           stage1_rank=c["stage1_rank"], stage2_tol=c["stage2_tol"], periodic=c["periodic"],
                           include_boundary=c["include_boundary"], qoi=f"p{ci}", provenance="golden pipeline")


def _sha(a):
    return np.frombuffer(hashlib.sha256(np.asfortranarray(a).tobytes(order="F")).digest(), dtype=np.uint8)


@pytest.mark.parametrize("ci", range(NCASES))
@pytest.mark.parametrize("per_push", [1, 3, 1000])
def test_pipeline_bytes_identical(PL, ci, per_push):
    c = _case(ci)
    data = PL.run_pipeline(c["a"], _cfg(PL, c, ci), frames_per_push=per_push)
    assert data == GOLD[f"pipe_{ci}_bytes"].tobytes()


@pytest.mark.parametrize("ci", range(NCASES))
def test_pipeline_device_frames(PL, ci):
    c = _case(ci)
    dev = torch.from_numpy(np.ascontiguousarray(c["a"].T)).cuda()  # row j = snapshot j
    with PL.Pipeline(_cfg(PL, c, ci)) as p:
        j = 0
        while j < c["n"]:  # uneven pushes of column-major device blocks
            cnt = min(1 + (j % 4), c["n"] - j)
            p.push(dev[j:j + cnt].T)
            j += cnt
        data = p.finish()
        st = p.stats()
    assert data == GOLD[f"pipe_{ci}_bytes"].tobytes()
    gst = GOLD[f"pipe_{ci}_stats"]
    assert st["snapshots"] == c["n"]
    assert st["stage1_tasks"] == gst[2] and st["stage2_tasks"] == gst[3]


@pytest.mark.parametrize("ci", range(NCASES))
def test_pipeline_decompress(PL, ci):
    from paper_2103_01380_b200 import archive as AR
    data = GOLD[f"pipe_{ci}_bytes"].tobytes()
    if f"pipe_{ci}_out_err" in GOLD.files:
        with pytest.raises(Exception) as e:
            AR.decompress(data)
        assert e.value.name == GOLD[f"pipe_{ci}_out_err"].tobytes().decode()
        return
    assert np.array_equal(_sha(AR.decompress(data)), GOLD[f"pipe_{ci}_out_sha"])
    info = json.loads(AR.archive_info_json(data))
    assert info["mode"] == "two-stage"


def test_pipeline_errors(PL):
    # stage-1 failure names block and chunk (test_pipeline.cpp:210-224)
    a = np.zeros((6, 4))
    a[0, 0] = 1.0
    a[1, 1] = 1.0
    cfg = PL.StreamConfig(dims=(6,), time_chunk=2, stage1_rank=1)
    with pytest.raises(Exception) as e:
        PL.run_pipeline(a, cfg)
    assert e.value.name == "ZeroMatrix"
    assert "block 0" in str(e.value) and "chunk 1" in str(e.value)
    # empty stream (test_pipeline.cpp:86-96)
    with PL.Pipeline(PL.StreamConfig(dims=(4,), time_chunk=2)) as p:
        with pytest.raises(Exception) as e:
            p.finish()
        assert e.value.name == "ShortStream"
    for kw, name in [(dict(time_chunk=0), "BadStreamConfig"), (dict(stage1_rank=0, time_chunk=2), "BadStreamConfig"),
                     (dict(blocks=(5,), time_chunk=2), "BlockTooSmall"),
                     (dict(strides=(0,), time_chunk=2), "BadSubsampleSpec")]:
        with pytest.raises(Exception) as e:
            PL.Pipeline(PL.StreamConfig(dims=(4,), **kw))
        assert e.value.name == name, (kw, e.value)
    with PL.Pipeline(PL.StreamConfig(dims=(4,), time_chunk=2)) as p:
        with pytest.raises(Exception) as e:
            p.push(np.ones(5))
        assert e.value.name == "GeometryMismatch"
    # stage-2 tolerance outside (0, 1) is raised by stage 2
    with PL.Pipeline(PL.StreamConfig(dims=(4,), time_chunk=2, stage2_tol=2.0)) as p:
        p.push(np.arange(8.0).reshape(4, 2) + 1.0)
        with pytest.raises(Exception) as e:
            p.finish()
        assert e.value.name == "BadRankRule"


def test_streaming_and_batch_agree(PL):
    """test_pipeline.cpp:226-234: stride 1, one chunk -> rank 3 on rank-3 data."""
    from paper_2103_01380_b200 import archive as AR
    rng = np.random.default_rng(77)
    a = rng.standard_normal((14, 3)) @ rng.standard_normal((3, 9))
    data = PL.run_pipeline(a, PL.StreamConfig(dims=(14,), time_chunk=9, stage1_rank=5))
    out = AR.decompress(data)
    assert np.linalg.norm(out - a) / np.linalg.norm(a) <= 1e-9
    assert json.loads(AR.archive_info_json(data))["block_ranks"] == [3]


def test_large_stream_vs_reference(PL, ref):
    """128^3 field, 64 blocks, 40 snapshots pushed one by one from the device,
    chunks of 16 (two full + one short): byte-identical to the reference."""
    g, n = 128, 40
    x = torch.linspace(0, 2 * torch.pi, g + 1, dtype=torch.float64, device="cuda")[:-1]
    X, Y, Z = torch.meshgrid(x, x, x, indexing="ij")
    frames = torch.stack([(torch.sin(X + 0.1 * j) * torch.cos(Y) * torch.cos(Z) +
                           0.2 * torch.cos(2 * X - 0.05 * j) * torch.sin(Y + Z)).permute(2, 1, 0).reshape(-1)
                          for j in range(n)])  # [n, m], x fastest
    frames += 1e-6 * torch.randn_like(frames)
    cfg = PL.StreamConfig(dims=(g,) * 3, blocks=(4, 4, 4), strides=(2, 2, 2), time_chunk=16, stage1_rank=6,
                          stage2_tol=1e-5, periodic=(1, 1, 1), qoi="u", provenance="large")
    with PL.Pipeline(cfg) as p:
        for j in range(n):
            p.push(frames[j])
        ours = p.finish()
    a = np.asfortranarray(frames.T.cpu().numpy())
    theirs, _ = ref.run_pipeline(a, (g,) * 3, (4, 4, 4), (2, 2, 2), 16, 6, 1e-5, periodic=(1, 1, 1), qoi="u",
                                 provenance="large")
    assert ours == theirs


def test_event_log_causality_and_counts(PL):
    """PipelineResult.events (proj/include/spid/pipeline.hpp:24-60): one
    SnapshotIngested per frame, ChunkClosed / Stage1Done per (block, chunk),
    Stage2Done per block; every chunk closes before its stage 1 completes and
    every stage 1 completes before stage 2 (proj/tests/test_pipeline.cpp:127)."""
    rng = np.random.default_rng(33)
    dims, blocks, T, n = (16, 12), (2, 2), 4, 14
    a = np.asfortranarray(rng.standard_normal((16 * 12, 2)) @ rng.standard_normal((2, n)))
    cfg = PL.StreamConfig(dims=dims, blocks=blocks, strides=(2, 2), time_chunk=T, stage1_rank=2, stage2_tol=1e-6)
    with PL.Pipeline(cfg) as p:
        for j in range(0, n, 3):
            p.push(a[:, j:j + 3])
        p.finish()
        ev = p.events()
    nb, nch = 4, -(-n // T)
    kinds = [e.kind for e in ev]
    assert kinds.count("SnapshotIngested") == n
    assert sorted(e.chunk for e in ev if e.kind == "SnapshotIngested") == list(range(n))
    assert kinds.count("ChunkClosed") == nb * nch and kinds.count("Stage1Done") == nb * nch
    assert kinds.count("Stage2Done") == nb
    closed = {(e.block, e.chunk): e.wall_time for e in ev if e.kind == "ChunkClosed"}
    done = {(e.block, e.chunk): e.wall_time for e in ev if e.kind == "Stage1Done"}
    stage2 = min(e.wall_time for e in ev if e.kind == "Stage2Done")
    assert set(closed) == set(done)
    for key, t in done.items():
        assert closed[key] <= t <= stage2
    for e in ev:
        assert e.duration >= 0.0 and e.wall_time >= e.duration
    rep = PL.overlap_report(ev)
    assert 0.0 <= rep["overlap_fraction"] <= 1.0 and rep["stage1_busy_seconds"] > 0.0
    # the reference's arithmetic on a hand-made log (pipeline.cpp:296-332)
    mk = lambda k, t, d: PL.TaskEvent(k, -1, 0, t, d)  # noqa: E731
    r = PL.overlap_report([mk("SnapshotIngested", 2.0, 1.0), mk("SnapshotIngested", 2.5, 1.0),
                           mk("SnapshotIngested", 5.0, 0.5), mk("Stage1Done", 3.0, 2.0)])
    assert r["producer_busy_seconds"] == pytest.approx(1.5 + 0.5)
    assert r["stage1_busy_seconds"] == pytest.approx(2.0)
    assert r["overlap_fraction"] == pytest.approx(1.5 / 2.0)
    with pytest.raises(PL.SpidError) as e:
        PL.overlap_report([])
    assert e.value.name == "EmptyLog"


def test_async_pushes_byte_identical():
    """Host frames pushed synchronously (on_device 0) and asynchronously from
    pinned memory (2: read in push order after the call returns, kept
    unmodified until finish), and device frames (1), give one archive."""
    import torch

    from paper_2103_01380_b200 import pipeline as PL

    g, T = 24, 5
    cfg = PL.StreamConfig(dims=(g, g, g), blocks=(2, 2, 2), strides=(2, 2, 2), time_chunk=T, stage1_rank=3,
                          stage2_tol=1e-6, periodic=(1, 1, 1), qoi="u", provenance="t")
    torch.manual_seed(3)
    n = 23
    x = torch.linspace(0, 6.283185307179586, g, dtype=torch.float64)
    base = (torch.sin(x)[:, None, None] * torch.cos(x)[None, :, None] * torch.cos(x)[None, None, :]).reshape(-1)
    frames = torch.stack([base * (0.9 ** t) + 1e-3 * torch.randn(base.shape, dtype=torch.float64)
                          for t in range(n)])  # [n, m]
    out = {}
    for name, src, sync in (("host", frames.numpy(), True), ("dev", frames.cuda(), True),
                            ("host_async", frames.pin_memory().numpy(), False)):
        with PL.Pipeline(cfg) as p:
            for j in range(n):
                p.push(src[j], sync=sync)
            out[name] = p.finish()
    assert out["host"] == out["dev"] == out["host_async"]
