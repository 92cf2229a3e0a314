"""ctypes binding of libspidgpu.so (include/spidgpu.h).

The library is the product: there is no Python or CPU implementation behind
these calls. If the .so is missing the import fails loudly; if no sm_100
device is present every handle creation raises SpidError("NoDevice").
"""
from __future__ import annotations

import ctypes as C
import os
import re
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# SPIDGPU_LIB_PATH: an alternative in-tree build (A/B experiments under tools/)
LIB_PATH = os.environ.get("SPIDGPU_LIB_PATH") or os.path.join(HERE, "lib", "libspidgpu.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "spidgpu.h")

RULE_FIXED, RULE_TOL, RULE_BLOCKED = 0, 1, 2
OMEGA_EXPLICIT, OMEGA_PHILOX = 0, 1
FIELD_TGV4, FIELD_TGV5, FIELD_MULTIMODE = 0, 1, 2
SPIDGPU_OPT_GENERIC_CPQR = 1
SPIDGPU_OPT_DMMA_SKETCH = 2
SPIDGPU_OPT_SKETCH_SMS = 4
SPIDGPU_OPT_SKETCH_PAIRS = 5
SPIDGPU_OPT_SKETCH_SEG_ROWS = 6
SPIDGPU_OPT_TALL_PAIRS = 7
SPIDGPU_OPT_REG_PAIRS = 8


class SpidError(RuntimeError):
    """Mirror of spid::Error (proj/include/spid/error.hpp:11-24): `name` is the
    reference's stable error name, the message follows after ': '."""

    def __init__(self, name: str, message: str = ""):
        super().__init__(f"{name}: {message}" if message else name)
        self.name = name


class RankRule(C.Structure):
    _fields_ = [("mode", C.c_int32), ("at_most", C.c_int32), ("k", C.c_int64),
                ("kstep", C.c_int64), ("tol", C.c_double)]


class Omega(C.Structure):
    _fields_ = [("mode", C.c_int32), ("reserved", C.c_int32), ("omega", C.c_void_p),
                ("ldo", C.c_int64), ("stride", C.c_int64), ("seed", C.c_uint64),
                ("subdomain_base", C.c_int64)]


class FieldSpec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_modes", C.c_int32), ("grid", C.c_int64),
                ("block", C.c_int64), ("snapshots", C.c_int64), ("t_end", C.c_double),
                ("nu", C.c_double), ("noise_sigma", C.c_double), ("kappa_max", C.c_double),
                ("mode_amp", C.c_double), ("seed", C.c_uint64), ("heavy_modes", C.c_int64),
                ("heavy_kmin", C.c_double)]


class GridSpec(C.Structure):
    _fields_ = [("naxes", C.c_int32), ("include_boundary", C.c_int32), ("dims", C.c_int64 * 3),
                ("strides", C.c_int64 * 3), ("periodic", C.c_int32 * 3), ("nqoi", C.c_int32)]


def grid_spec(dims, strides, periodic=None, include_boundary=True, nqoi=1) -> GridSpec:
    nax = len(dims)
    per = [int(bool(x)) for x in periodic] if periodic else [0] * nax
    pad = lambda v, f: list(v) + [f] * (3 - nax)  # noqa: E731
    return GridSpec(nax, int(bool(include_boundary)), (C.c_int64 * 3)(*pad(dims, 1)),
                    (C.c_int64 * 3)(*pad(strides, 1)), (C.c_int32 * 3)(*pad(per, 0)), nqoi)


ARCHIVE_EXACT, ARCHIVE_SKETCH = 0, 1


class ArchiveSpec(C.Structure):
    _fields_ = [("naxes", C.c_int32), ("mode", C.c_int32), ("dims", C.c_int64 * 3),
                ("periodic", C.c_int32 * 3), ("reserved", C.c_int32),
                ("blocks_per_axis", C.c_int64 * 3), ("strides", C.c_int64 * 3),
                ("ell", C.c_int64), ("seed", C.c_uint64), ("qoi", C.c_char_p),
                ("provenance", C.c_char_p)]


def archive_spec(dims, blocks, strides, periodic=None, mode=ARCHIVE_EXACT, ell=0, seed=0,
                 qoi="", provenance="") -> ArchiveSpec:
    nax = len(dims)
    per = [int(bool(x)) for x in periodic] if periodic else [0] * nax
    pad = lambda v, f: list(v) + [f] * (3 - nax)  # noqa: E731
    return ArchiveSpec(nax, mode, (C.c_int64 * 3)(*pad(dims, 1)), (C.c_int32 * 3)(*pad(per, 0)), 0,
                       (C.c_int64 * 3)(*pad(blocks, 1)), (C.c_int64 * 3)(*pad(strides, 1)), ell,
                       seed, qoi.encode(), provenance.encode())


class StreamConfig(C.Structure):
    _fields_ = [("naxes", C.c_int32), ("include_boundary", C.c_int32), ("dims", C.c_int64 * 3),
                ("periodic", C.c_int32 * 3), ("reserved", C.c_int32),
                ("blocks_per_axis", C.c_int64 * 3), ("strides", C.c_int64 * 3),
                ("time_chunk", C.c_int64), ("stage1_rank", C.c_int64), ("stage2_tol", C.c_double),
                ("qoi", C.c_char_p), ("provenance", C.c_char_p)]


class StreamStats(C.Structure):
    _fields_ = [("snapshots", C.c_int64), ("stage1_tasks", C.c_int64), ("stage2_tasks", C.c_int64),
                ("fine_entries_peak", C.c_int64), ("coarse_entries_peak", C.c_int64),
                ("stage1_ms", C.c_double), ("stage2_ms", C.c_double)]


class TaskEvent(C.Structure):
    _fields_ = [("kind", C.c_int32), ("block", C.c_int64), ("chunk", C.c_int64), ("wall_time", C.c_double),
                ("duration", C.c_double)]


class Overlap(C.Structure):
    _fields_ = [("overlap_fraction", C.c_double), ("stage1_busy_seconds", C.c_double),
                ("producer_busy_seconds", C.c_double)]


EVENT_KINDS = ("SnapshotIngested", "ChunkClosed", "Stage1Done", "Stage2Done")

_vp = C.c_void_p
_i64 = C.c_int64
_H = C.c_void_p
_RR = C.POINTER(RankRule)
_OM = C.POINTER(Omega)
_GS = C.POINTER(GridSpec)
_AS = C.POINTER(ArchiveSpec)
_pi64 = C.POINTER(C.c_int64)

# name -> (restype, argtypes)
_SIGS = {
    "spidgpu_create": (C.c_int, [C.c_int, C.POINTER(_H)]),
    "spidgpu_destroy": (C.c_int, [_H]),
    "spidgpu_status_name": (C.c_char_p, [C.c_int]),
    "spidgpu_last_error": (C.c_char_p, [_H]),
    "spidgpu_abi_version": (C.c_int, []),
    "spidgpu_launch_count": (C.c_int64, [_H]),
    "spidgpu_set_option": (C.c_int, [_H, C.c_int, C.c_int64]),
    "spidgpu_stream_status": (C.c_int, [_H, _vp]),
    "spidgpu_reserve": (C.c_int, [_H, _i64, _i64, _i64, _i64, _i64]),
    "spidgpu_debug_counters": (C.c_int, [_H, C.POINTER(C.c_int64), C.c_int, C.c_int]),
    "spidgpu_sketch_batched": (C.c_int, [_H, _vp, _i64, _i64, _i64, _i64, _i64, _i64, _OM, _vp,
                                         _i64, _i64, _vp]),
    "spidgpu_philox_omega": (C.c_int, [_H, C.c_uint64, _i64, _i64, _i64, _vp, _i64, _vp]),
    "spidgpu_cpqr_id_batched": (C.c_int, [_H, _vp, _i64, _i64, _i64, _i64, _i64, _RR, _i64, _vp,
                                          _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "spidgpu_gather_batched": (C.c_int, [_H, _vp, _i64, _i64, _i64, _i64, _i64, _vp, _i64, _vp,
                                         _vp, _i64, _i64, _vp]),
    "spidgpu_row_gather_batched": (C.c_int, [_H, _vp, _i64, _i64, _i64, _i64, _i64, _vp, _i64,
                                             _vp, _i64, _i64, _vp]),
    "spidgpu_verify_batched": (C.c_int, [_H, _vp, _i64, _i64, _i64, _i64, _i64, _vp, _i64, _i64,
                                         _vp, _i64, _i64, _vp, _vp, _vp, _vp]),
    "spidgpu_reconstruct_batched": (C.c_int, [_H, _vp, _i64, _i64, _i64, _vp, _i64, _i64, _vp,
                                              _i64, _i64, _vp, _i64, _i64, _vp]),
    "spidgpu_compress_batched": (C.c_int, [_H, _vp, _i64, _i64, _i64, _i64, _i64, _i64, _OM, _RR,
                                           _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "spidgpu_column_id": (C.c_int, [_H, _vp, _i64, _i64, _RR, _i64, _vp, _vp, _vp, _vp, _vp]),
    "spidgpu_qr": (C.c_int, [_H, _vp, _i64, _i64, _RR, _i64, _vp, _vp, _vp, _vp, _vp]),
    "spidgpu_sub_id": (C.c_int, [_H, _vp, _i64, _i64, _vp, _i64, _RR, _i64, _vp, _vp, _vp, _vp,
                                 _vp]),
    "spidgpu_sketch_id": (C.c_int, [_H, _vp, _i64, _i64, _i64, _OM, _RR, _i64, _vp, _vp, _vp, _vp,
                                    _vp, _vp]),
    "spidgpu_reconstruct": (C.c_int, [_H, _vp, _i64, _i64, _vp, _i64, _vp]),
    "spidgpu_rel_frob_error": (C.c_int, [_H, _vp, _vp, _i64, _i64, C.POINTER(C.c_double)]),
    "spidgpu_compression_factor": (C.c_int, [_i64, _i64, _i64, C.POINTER(C.c_double)]),
    "spidgpu_compress_host": (C.c_int, [_H, _vp, _i64, _i64, _i64, _i64, _OM, _RR, _i64, _i64,
                                        _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "spidgpu_crc32": (C.c_int, [_H, _vp, _i64, C.c_int32, C.POINTER(C.c_uint32)]),
    "spidgpu_archive_compress": (C.c_int, [_H, _vp, _i64, _i64, _i64, C.c_int32, _AS, _RR, _pi64]),
    "spidgpu_archive_fetch": (C.c_int, [_H, _vp, _i64]),
    "spidgpu_archive_view": (C.c_int, [_H, C.POINTER(_vp), _pi64]),
    "spidgpu_archive_shape": (C.c_int, [_vp, _i64, _pi64, _pi64, _pi64]),
    "spidgpu_archive_info": (C.c_int, [_H, _vp, _i64, _vp, _i64, _pi64]),
    "spidgpu_archive_decompress": (C.c_int, [_H, _vp, _i64, _vp, _i64, C.c_int32]),
    "spidgpu_stream_open": (C.c_int, [_H, C.POINTER(StreamConfig), C.POINTER(_vp)]),
    "spidgpu_stream_push": (C.c_int, [_vp, _vp, _i64, _i64, _i64, C.c_int32]),
    "spidgpu_stream_finish": (C.c_int, [_vp, _pi64]),
    "spidgpu_stream_get_stats": (C.c_int, [_vp, C.POINTER(StreamStats)]),
    "spidgpu_stream_events": (C.c_int, [_vp, C.POINTER(TaskEvent), _i64, C.POINTER(C.c_int64)]),
    "spidgpu_overlap_report": (C.c_int, [C.POINTER(TaskEvent), _i64, C.POINTER(Overlap)]),
    "spidgpu_stream_last_error": (C.c_char_p, [_vp]),
    "spidgpu_stream_close": (C.c_int, [_vp]),
    "spidgpu_field_generate": (C.c_int, [_H, C.POINTER(FieldSpec), _i64, _i64, _vp, _vp, _i64,
                                         _i64, _vp]),
    "spidgpu_row_indices": (C.c_int, [_GS, _vp, _i64, C.POINTER(C.c_int64)]),
    "spidgpu_spid": (C.c_int, [_H, _vp, _i64, _i64, _GS, _RR, _i64, _vp, _vp, _vp, _vp, _vp]),
    "spidgpu_interp_apply": (C.c_int, [_H, _GS, _vp, _i64, _i64, _vp]),
    "spidgpu_spid_reconstruct": (C.c_int, [_H, _GS, _vp, _i64, _i64, _vp, _i64, _i64, _vp]),
    "spidgpu_gather_coarse_batched": (C.c_int, [_H, _vp, _i64, _i64, _i64, _i64, _i64, _GS, _vp,
                                                _i64, _vp, _vp, _i64, _i64, _vp]),
    "spidgpu_interp_apply_batched": (C.c_int, [_H, _GS, _vp, _i64, _i64, _i64, _vp, _i64, _vp,
                                               _i64, _i64, _vp]),
}


def header_symbols(path: str = HEADER) -> list[str]:
    """Every function the C ABI header declares."""
    text = open(path).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(spidgpu_\w+)\s*\(", text,
                                 re.M)))


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_2103_01380_b200.build`"
                          " (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        if os.environ.get("SPIDGPU_LIB_PATH") and not hasattr(lib, name):
            continue  # an older A/B build may predate newer entry points
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def status_name(code: int) -> str:
    return lib.spidgpu_status_name(code).decode()


class Handle:
    """One spidgpu handle (device context + workspaces). Not thread-safe:
    use one per host thread / stream, like the ABI says."""

    def __init__(self, device: int = 0):
        h = _H()
        rc = lib.spidgpu_create(device, C.byref(h))
        if rc:
            raise SpidError(status_name(rc), f"spidgpu_create(device={device}) failed")
        self.h = h
        self.device = device

    def check(self, rc: int):
        if rc:
            raise SpidError(status_name(rc), lib.spidgpu_last_error(self.h).decode())

    def launches(self) -> int:
        return lib.spidgpu_launch_count(self.h)

    def close(self):
        if getattr(self, "h", None):
            lib.spidgpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_local = threading.local()


def handle(device: int = 0) -> Handle:
    """Per-thread, per-device cached handle."""
    cache = getattr(_local, "handles", None)
    if cache is None:
        cache = _local.handles = {}
    if device not in cache:
        cache[device] = Handle(device)
    return cache[device]
