"""Streaming two-stage compressor: the reference's spid/pipeline.hpp surface
(StreamConfig, run_pipeline -- proj/include/spid/pipeline.hpp,
proj/src/pipeline.cpp:104-294) over the C ABI's spidgpu_stream_* calls.

    cfg = StreamConfig(dims=(64, 64, 64), blocks=(4, 4, 4), strides=(2, 2, 2),
                       time_chunk=16, stage1_rank=8, stage2_tol=1e-6)
    with Pipeline(cfg) as p:
        for frame in solver:          # one m-vector (numpy or CUDA tensor) per step
            p.push(frame)
        data = p.finish()             # == encode(run_pipeline(producer, cfg).archive)

Snapshots never leave the GPU once pushed: each block's coarse rows are
buffered in device chunks, stage 1 runs per closed chunk on a second CUDA
stream, stage 2 and the archive at finish.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from ._native import SpidError

__all__ = ["StreamConfig", "Pipeline", "run_pipeline", "TaskEvent", "overlap_report"]


@dataclass
class TaskEvent:
    """spid::TaskEvent (proj/include/spid/pipeline.hpp:24-32); times in
    seconds on the device timeline from the stream's open."""
    kind: str       # SnapshotIngested | ChunkClosed | Stage1Done | Stage2Done
    block: int
    chunk: int
    wall_time: float
    duration: float


def overlap_report(events) -> dict:
    """spid::overlap_report (proj/src/pipeline.cpp:296-332): the fraction of
    stage-1 time that ran while ingestion was busy."""
    arr = (N.TaskEvent * max(1, len(events)))()
    for i, e in enumerate(events):
        arr[i] = N.TaskEvent(N.EVENT_KINDS.index(e.kind), e.block, e.chunk, e.wall_time, e.duration)
    out = N.Overlap()
    rc = N.lib.spidgpu_overlap_report(arr, len(events), C.byref(out))
    if rc:
        raise SpidError(N.status_name(rc), "overlap_report")
    return {k: getattr(out, k) for k, _ in N.Overlap._fields_}


@dataclass
class StreamConfig:
    """spid::StreamConfig + PartitionPlan (pipeline.hpp:14-24, blocking.hpp)."""
    dims: tuple
    blocks: tuple | None = None
    strides: tuple | None = None
    time_chunk: int = 1
    stage1_rank: int = 1
    stage2_tol: float = 1e-6
    periodic: tuple | None = None
    include_boundary: bool = True
    qoi: str = ""
    provenance: str = ""

    def c(self) -> N.StreamConfig:
        nax = len(self.dims)
        pad = lambda v, f: list(v) + [f] * (3 - nax)  # noqa: E731
        blocks = self.blocks or [1] * nax
        strides = self.strides or [1] * nax
        per = [int(bool(x)) for x in self.periodic] if self.periodic else [0] * nax
        return N.StreamConfig(nax, int(bool(self.include_boundary)), (C.c_int64 * 3)(*pad(self.dims, 2)),
                              (C.c_int32 * 3)(*pad(per, 0)), 0, (C.c_int64 * 3)(*pad(blocks, 1)),
                              (C.c_int64 * 3)(*pad(strides, 1)), self.time_chunk, self.stage1_rank,
                              self.stage2_tol, self.qoi.encode(), self.provenance.encode())


class Pipeline:
    """One streaming compression (run_pipeline) on a device."""

    def __init__(self, config: StreamConfig, device: int = 0):
        self.h = N.handle(device)
        self._cfg = config.c()  # keeps the metadata strings alive
        s = C.c_void_p()
        self.h.check(N.lib.spidgpu_stream_open(self.h.h, C.byref(self._cfg), C.byref(s)))
        self.s = s
        self.m = int(np.prod(config.dims))

    def _check(self, rc):
        if rc:
            raise SpidError(N.status_name(rc), N.lib.spidgpu_stream_last_error(self.s).decode())

    def push(self, frames, *, sync: bool = True):
        """Push one frame (m,) or a block of frames (m, count): numpy (host)
        or a CUDA tensor in column-major layout. CUDA frames are read
        asynchronously: keep them unmodified until finish(). Host frames:
        sync=True copies them before the call returns; sync=False reads them
        asynchronously too (keep them alive and unmodified until finish();
        pinned memory, e.g. a pinned torch tensor's .numpy(), lets the copies
        overlap)."""
        if hasattr(frames, "is_cuda") and frames.is_cuda:
            f = frames if frames.dim() == 2 else frames.reshape(-1, 1)
            if f.shape[1] > 1 and f.stride(0) != 1:
                raise ValueError("device frames must be column-major (frames.T contiguous)")
            m, cnt = f.shape
            ld = f.stride(1) if cnt > 1 else m
            self._check(N.lib.spidgpu_stream_push(self.s, C.c_void_p(f.data_ptr()), m, cnt, ld, 1))
            return
        f = np.asfortranarray(np.asarray(frames, dtype=np.float64))
        if f.ndim == 1:
            f = f.reshape(-1, 1, order="F")
        m, cnt = f.shape
        if not sync and not (isinstance(frames, np.ndarray) and np.may_share_memory(f, frames)):
            raise ValueError("sync=False needs host frames the stream can read in place (float64, column-major)")
        self._check(N.lib.spidgpu_stream_push(self.s, C.c_void_p(f.ctypes.data), m, cnt, max(m, 1), 0 if sync else 2))

    def finish(self) -> bytes:
        nb = C.c_int64()
        self._check(N.lib.spidgpu_stream_finish(self.s, C.byref(nb)))
        view, n = C.c_void_p(), C.c_int64()
        self.h.check(N.lib.spidgpu_archive_view(self.h.h, C.byref(view), C.byref(n)))
        return C.string_at(view.value, n.value)

    def stats(self) -> dict:
        st = N.StreamStats()
        self._check(N.lib.spidgpu_stream_get_stats(self.s, C.byref(st)))
        return {k: getattr(st, k) for k, _ in N.StreamStats._fields_}

    def events(self) -> list:
        """The event log (PipelineResult.events) -- after finish()."""
        n = C.c_int64()
        self._check(N.lib.spidgpu_stream_events(self.s, None, 0, C.byref(n)))
        arr = (N.TaskEvent * max(1, n.value))()
        self._check(N.lib.spidgpu_stream_events(self.s, arr, n.value, C.byref(n)))
        return [TaskEvent(N.EVENT_KINDS[e.kind], e.block, e.chunk, e.wall_time, e.duration)
                for e in arr[:n.value]]

    def close(self):
        if getattr(self, "s", None):
            N.lib.spidgpu_stream_close(self.s)
            self.s = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_pipeline(a, config: StreamConfig, *, frames_per_push: int = 1, device: int = 0) -> bytes:
    """run_pipeline(MatrixProducer(a), config) -> encoded archive: the columns
    of `a` (m x n) are pushed `frames_per_push` at a time, in time order."""
    with Pipeline(config, device) as p:
        n = a.shape[1]
        for j in range(0, n, frames_per_push):
            p.push(a[:, j:j + frames_per_push])
        return p.finish()
