"""CPU oracle for the SPID compression path -- TEST INFRASTRUCTURE ONLY.

Two checkers behind one numpy-facing interface:

* ``port`` -- ``oracle/spid_oracle.c``, a plain-C restatement of the
  reference (every function cites the reference file:line it follows);
* ``ref``  -- the reference itself (``/root/reference/proj/src``) compiled by
  ``oracle/Makefile`` into ``oracle/_ref/libspidref.so``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this package. The product path
(``paper_2103_01380_b200``) never imports it and has no CPU fallback.

Matrices are numpy arrays; column-major (Fortran) order is used throughout to
match the reference's DenseMatrix (proj/include/spid/dense_matrix.hpp:33-34).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libspid_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspidref.so")

RULE_FIXED, RULE_TOL, RULE_BLOCKED = 0, 1, 2

STATUS_NAMES = {
    0: "Ok", 1: "NonFiniteInput", 2: "RankUnreachable", 3: "ZeroMatrix",
    4: "SingularPivot", 5: "DimensionMismatch", 6: "NonFiniteCoeffs",
    7: "BadRankRule", 8: "EmptyMatrix", 9: "EmptySelection",
    10: "IndexOutOfRange", 11: "GeometryMismatch", 12: "ZeroReference",
    13: "ZeroDenominator", 14: "BadSubsampleSpec", 15: "EmptySketch", 16: "ExtrapolationRequired", 17: "BadGridGeom",
    18: "BlockTooSmall", 19: "BadMagic", 20: "VersionUnsupported", 21: "TruncatedPayload",
    22: "ChecksumMismatch", 23: "CoverageGap", 24: "UnstructuredNoInterp", 25: "BadStreamConfig", 26: "ShortStream", 27: "EmptyLog",
    100: "CudaError", 101: "InvalidArgument", 102: "ShapeUnsupported", 103: "NoDevice",
}


class OracleError(RuntimeError):
    """Mirrors spid::Error: carries the reference's stable error name."""

    def __init__(self, name: str):
        super().__init__(name)
        self.name = name


def build(quiet: bool = True) -> None:
    """Compile the oracle (and _ref when /root/reference is present)."""
    subprocess.run(["make", "-C", HERE, "all"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)
_SZ = C.POINTER(C.c_size_t)
_sz = C.c_size_t


def _dp(a):
    return a.ctypes.data_as(_D) if a is not None else None


def _ip(a):
    return a.ctypes.data_as(_I64) if a is not None else None


def _f64(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


@dataclass
class IdResult:
    """Mirror of spid::IdFactors (proj/include/spid/id.hpp:12-19)."""
    indices: np.ndarray   # (rank,) selection order
    coeffs: np.ndarray    # (rank, n) Fortran
    skeleton: np.ndarray | None  # (m, rank) Fortran
    rank: int
    residual_fro: float
    y: np.ndarray | None = None  # the sketch, when one was formed


@dataclass
class QrResult:
    """Mirror of spid::QrFactorization (proj/include/spid/qr.hpp:45-51)."""
    q: np.ndarray
    r: np.ndarray
    pivots: np.ndarray
    rank: int
    residual_fro: float


def _rule_args(rank, tol, kstep=None):
    if kstep is not None:
        return RULE_BLOCKED, int(rank), float(tol), int(kstep)
    if (rank is None) == (tol is None):
        raise ValueError("pass exactly one of rank= or tol=")
    if rank is not None:
        return RULE_FIXED, int(rank), 0.0, 0
    return RULE_TOL, 0, float(tol), 0


class _FieldSpec(C.Structure):
    """orc_field_spec == spidgpu_field_spec (include/spidgpu.h)."""
    _fields_ = [("kind", C.c_int32), ("n_modes", C.c_int32), ("grid", C.c_int64), ("block", C.c_int64),
                ("snapshots", C.c_int64), ("t_end", C.c_double), ("nu", C.c_double), ("sigma", C.c_double),
                ("kappa_max", C.c_double), ("mode_amp", C.c_double), ("seed", C.c_uint64),
                ("heavy_modes", C.c_int64), ("heavy_kmin", C.c_double)]


class _Port:
    """The C restatement (oracle/spid_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.orc_seeded_sym.argtypes = [C.c_uint64, _D, _sz]
        L.orc_gaussian.argtypes = [C.c_uint64, _D, _sz]
        L.orc_splitmix_next.argtypes = [C.POINTER(C.c_uint64)]
        L.orc_splitmix_next.restype = C.c_uint64
        L.orc_matmul.argtypes = [_D, _sz, _sz, _D, _sz, _D]
        L.orc_frobenius.argtypes = [_D, _sz]
        L.orc_frobenius.restype = C.c_double
        L.orc_qr.argtypes = [_D, _sz, _sz, C.c_int, _sz, C.c_double, _sz, C.c_int, _sz,
                             _D, _D, _I64, _SZ, _D]
        L.orc_solve_upper.argtypes = [_D, _sz, _sz, _D, _sz, _D]
        L.orc_column_id.argtypes = [_D, _sz, _sz, C.c_int, _sz, C.c_double, _sz, C.c_int, _sz,
                                    _I64, _D, _D, _SZ, _D]
        L.orc_sketch_id.argtypes = [_D, _sz, _sz, _D, _sz, C.c_int, _sz, C.c_double, _sz, _sz,
                                    _D, _I64, _D, _D, _SZ, _D]
        L.orc_error_terms.argtypes = [_D, _sz, _sz, _D, _sz, _D, _sz, _sz, _D, _D]
        L.orc_rel_frob_error.argtypes = [_D, _D, _sz, _D]
        L.orc_compression_factor.argtypes = [_sz, _sz, _sz, _D]
        L.orc_row_indices.argtypes = [_SZ, C.POINTER(C.c_int), _SZ, _sz, C.c_int, _I64, _sz, _SZ]
        L.orc_interp_apply.argtypes = [_SZ, C.POINTER(C.c_int), _SZ, _sz, C.c_int, _D, _sz, _D]
        L.orc_omega_table.argtypes = [C.c_void_p]
        L.orc_philox_omega.argtypes = [C.c_uint64, C.c_uint64, _sz, _sz, _sz, _D]
        L.orc_field_generate.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, _D, C.c_int64,
                                         C.c_int64, C.c_int]
        self.lib = L

    # ---- workload generation (oracle/workload.c) -------------------------------
    def omega_table(self) -> np.ndarray:
        q = np.zeros(4096, dtype=np.int8)
        self.lib.orc_omega_table(q.ctypes.data_as(C.c_void_p))
        return q

    def philox_omega(self, seed, s, ell, m, row0=0) -> np.ndarray:
        """Omega_s rows [row0, row0+ell) as an (ell, m) Fortran array -- the
        matrix the in-kernel Philox sketch contracts."""
        out = np.zeros((ell, m), dtype=np.float64, order="F")
        self.lib.orc_philox_omega(int(seed), int(s), int(row0), int(ell), int(m), _dp(out))
        return out

    def field_generate(self, spec: dict, first, batch, is_heavy=None, threads=None, out=None) -> np.ndarray:
        """Subdomains [first, first+batch) of a BASELINE synthetic field as a
        (batch, n, m) array (= batch column-major m x n matrices). spec holds
        the spidgpu_field_spec fields (paper_2103_01380_b200/configs.py)."""
        fs = _FieldSpec(**spec)
        nq = 4 if fs.kind == 0 else 5
        m, n = nq * fs.block ** 3, fs.snapshots
        a = out if out is not None else np.empty((batch, n, m), dtype=np.float64)
        hv = None
        if is_heavy is not None:
            hv = np.ascontiguousarray(is_heavy, dtype=np.uint8)
        rc = self.lib.orc_field_generate(C.byref(fs), int(first), int(batch),
                                         hv.ctypes.data_as(C.c_void_p) if hv is not None else None,
                                         _dp(a), m, m * n, int(threads or os.cpu_count() or 1))
        self._check(rc)
        return a

    @staticmethod
    def _spec(dims, strides, periodic):
        nax = len(dims)
        return ((C.c_size_t * nax)(*dims), (C.c_int * nax)(*([int(bool(x)) for x in periodic]
                                                               if periodic else [0] * nax)),
                (C.c_size_t * nax)(*strides), nax)

    def row_indices(self, dims, strides, periodic=None, include_boundary=True):
        d, p, s, nax = self._spec(dims, strides, periodic)
        cap = int(np.prod(dims))
        out = np.zeros(cap, dtype=np.int64)
        cnt = C.c_size_t(0)
        self._check(self.lib.orc_row_indices(d, p, s, nax, int(include_boundary), _ip(out), cap,
                                             C.byref(cnt)))
        return out[:cnt.value].copy()

    def interp_apply(self, dims, strides, coarse, periodic=None, include_boundary=True):
        """InterpOperator::from_spec(spec).apply(coarse) (interp.cpp:45-100, 168-186)."""
        d, p, s, nax = self._spec(dims, strides, periodic)
        coarse = _f64(coarse)
        fine = np.zeros((int(np.prod(dims)), coarse.shape[1]), order="F")
        self._check(self.lib.orc_interp_apply(d, p, s, nax, int(include_boundary), _dp(coarse),
                                              coarse.shape[1], _dp(fine)))
        return fine

    @staticmethod
    def _check(st):
        if st:
            raise OracleError(STATUS_NAMES.get(st, f"status{st}"))

    def seeded_matrix(self, m, n, seed):
        """proj/tests/common.hpp:13-19 (SplitMix64 next_sym, column-major)."""
        out = np.empty((m, n), dtype=np.float64, order="F")
        self.lib.orc_seeded_sym(seed, _dp(out), m * n)
        return out

    def splitmix_next(self, state: list) -> int:
        """SplitMix64::next_u64 on a one-element list holding the state."""
        st = C.c_uint64(state[0])
        v = self.lib.orc_splitmix_next(C.byref(st))
        state[0] = st.value
        return int(v)

    def seeded_vector(self, m, seed):
        out = np.empty(m, dtype=np.float64)
        self.lib.orc_seeded_sym(seed, _dp(out), m)
        return out

    def gaussian(self, rows, cols, seed):
        out = np.empty((rows, cols), dtype=np.float64, order="F")
        self.lib.orc_gaussian(seed, _dp(out), rows * cols)
        return out

    def matmul(self, a, b):
        a, b = _f64(a), _f64(b)
        assert a.shape[1] == b.shape[0]
        c = np.empty((a.shape[0], b.shape[1]), dtype=np.float64, order="F")
        self.lib.orc_matmul(_dp(a), a.shape[0], a.shape[1], _dp(b), b.shape[1], _dp(c))
        return c

    def frobenius(self, a):
        a = _f64(a)
        return self.lib.orc_frobenius(_dp(a), a.size)

    def qr(self, a, rank=None, tol=None, at_most=False, kstep=None):
        a = _f64(a)
        m, n = a.shape
        mode, k, t, ks = _rule_args(rank, tol, kstep)
        if at_most:
            k = max(1, min(k, m, n))
        kcap = max(1, min(m, n) if mode == RULE_TOL else min(k, min(m, n)))
        q = np.zeros((m, kcap), order="F")
        r = np.zeros((kcap, n), order="F")
        piv = np.zeros(n, dtype=np.int64)
        rank_out = C.c_size_t(0)
        res = C.c_double(0)
        self._check(self.lib.orc_qr(_dp(a), m, n, mode, k, t, ks, 0 if at_most else 1, kcap,
                                    _dp(q), _dp(r), _ip(piv), C.byref(rank_out), C.byref(res)))
        rk = rank_out.value
        return QrResult(np.asfortranarray(q[:, :rk]), np.asfortranarray(r[:rk, :]), piv, rk,
                        res.value)

    def solve_upper(self, r11, rhs):
        r11, rhs = _f64(r11), _f64(rhs)
        k = r11.shape[0]
        x = np.empty_like(rhs, order="F")
        self._check(self.lib.orc_solve_upper(_dp(r11), k, k, _dp(rhs), rhs.shape[1], _dp(x)))
        return x

    def column_id(self, a, rank=None, tol=None, at_most=False, kstep=None):
        a = _f64(a)
        m, n = a.shape
        mode, k, t, ks = _rule_args(rank, tol, kstep)
        kcap = max(1, min(m, n))
        idx = np.zeros(kcap, dtype=np.int64)
        coeffs = np.zeros((kcap, n), order="F")
        skel = np.zeros((m, kcap), order="F")
        rank_out = C.c_size_t(0)
        res = C.c_double(0)
        self._check(self.lib.orc_column_id(_dp(a), m, n, mode, k, t, ks, 1 if at_most else 0,
                                           kcap, _ip(idx), _dp(coeffs), _dp(skel),
                                           C.byref(rank_out), C.byref(res)))
        rk = rank_out.value
        return IdResult(idx[:rk].copy(), np.asfortranarray(coeffs[:rk]),
                        np.asfortranarray(skel[:, :rk]), rk, res.value)

    def sketch_id(self, a, omega, rank=None, tol=None, kstep=None, want_y=True):
        """Gaussian-sketch SubID: the BASELINE north-star path on the CPU."""
        a, omega = _f64(a), _f64(omega)
        m, n = a.shape
        ell = omega.shape[0]
        assert omega.shape[1] == m
        mode, k, t, ks = _rule_args(rank, tol, kstep)
        kcap = max(1, min(ell, n))
        y = np.zeros((ell, n), order="F") if want_y else None
        idx = np.zeros(kcap, dtype=np.int64)
        coeffs = np.zeros((kcap, n), order="F")
        skel = np.zeros((m, kcap), order="F")
        rank_out = C.c_size_t(0)
        res = C.c_double(0)
        self._check(self.lib.orc_sketch_id(_dp(a), m, n, _dp(omega), ell, mode, k, t, ks, kcap,
                                           _dp(y), _ip(idx), _dp(coeffs), _dp(skel),
                                           C.byref(rank_out), C.byref(res)))
        rk = rank_out.value
        return IdResult(idx[:rk].copy(), np.asfortranarray(coeffs[:rk]),
                        np.asfortranarray(skel[:, :rk]), rk, res.value, y)

    def error_terms(self, a, skeleton, coeffs):
        """(||A - S C||_F^2, ||A||_F^2) by the reference's route."""
        a, s, c = _f64(a), _f64(skeleton), _f64(coeffs)
        e2, r2 = C.c_double(0), C.c_double(0)
        self._check(self.lib.orc_error_terms(_dp(a), a.shape[0], a.shape[1], _dp(s), s.shape[0],
                                             _dp(c), c.shape[0], c.shape[0], C.byref(e2),
                                             C.byref(r2)))
        return e2.value, r2.value

    def rel_frob_error(self, exact, approx):
        exact, approx = _f64(exact), _f64(approx)
        if exact.shape != approx.shape:
            raise OracleError("DimensionMismatch")
        out = C.c_double(0)
        self._check(self.lib.orc_rel_frob_error(_dp(exact), _dp(approx), exact.size,
                                                C.byref(out)))
        return out.value

    def compression_factor(self, m, n, stored):
        out = C.c_double(0)
        self._check(self.lib.orc_compression_factor(m, n, stored, C.byref(out)))
        return out.value


class _Ref:
    """The reference compiled from /root/reference (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        cp = C.c_char_p
        L.ref_matmul.argtypes = [_D, _sz, _sz, _D, _sz, _D, cp, _sz]
        L.ref_qr.argtypes = [_D, _sz, _sz, C.c_int, _sz, C.c_double, C.c_int, _sz, _D, _D, _I64,
                             _SZ, _D, cp, _sz]
        L.ref_column_id.argtypes = [_D, _sz, _sz, C.c_int, _sz, C.c_double, C.c_int, _sz, _I64,
                                    _D, _D, _SZ, _D, cp, _sz]
        L.ref_sub_id.argtypes = [_D, _sz, _sz, _SZ, C.POINTER(C.c_int), _SZ, _sz, C.c_int, _sz,
                                 C.c_double, _sz, _I64, _D, _D, _SZ, _D, cp, _sz]
        L.ref_row_indices.argtypes = [_SZ, C.POINTER(C.c_int), _SZ, _sz, _I64, _sz, _SZ, cp, _sz]
        L.ref_rel_frob_error.argtypes = [_D, _D, _sz, _sz, _D, cp, _sz]
        L.ref_compression_factor.argtypes = [_sz, _sz, _sz, _D, cp, _sz]
        L.ref_compress_batch.argtypes = [_D, _sz, _sz, _sz, _D, _sz, _sz, C.c_int, _SZ, _D, cp,
                                         _sz]
        L.ref_spid.argtypes = [_D, _sz, _sz, _SZ, C.POINTER(C.c_int), _SZ, _sz, C.c_int, C.c_int,
                               _sz, C.c_double, _sz, _I64, _D, _D, _D, _SZ, _D, cp, _sz]
        L.ref_interp_apply.argtypes = [_SZ, C.POINTER(C.c_int), _SZ, _sz, C.c_int, _D, _sz, _D,
                                       cp, _sz]
        L.ref_compress_field.argtypes = [_D, _sz, _sz, _SZ, C.POINTER(C.c_int), _sz, _SZ, _SZ, _sz,
                                         C.c_double, cp, cp, _SZ, cp, _sz]
        L.ref_archive_fetch.argtypes = [C.c_void_p, _sz]
        L.ref_archive_decompress.argtypes = [C.c_void_p, _sz, _D, _sz, _SZ, _SZ, cp, _sz]
        L.ref_archive_info.argtypes = [C.c_void_p, _sz, cp, _sz, cp, _sz]
        L.ref_crc32.argtypes = [C.c_void_p, _sz]
        L.ref_crc32.restype = C.c_uint32
        self.lib = L

    # ---- archive codec (proj/src/archive.cpp; CLI batch compress) ----------------
    def compress_field(self, a, dims, blocks, strides, rank=0, tol=0.0, periodic=None, qoi="",
                       provenance=""):
        """The CLI's batch compression of a structured field + encode() -> bytes."""
        a = _f64(a)
        m, n = a.shape
        nax = len(dims)
        d, p, s, _ = _Port._spec(dims, strides, periodic)
        b = (C.c_size_t * nax)(*blocks)
        nb = C.c_size_t(0)
        self._call(self.lib.ref_compress_field, _dp(a), m, n, d, p, nax, b, s, int(rank or 0),
                   float(tol or 0.0), qoi.encode(), provenance.encode(), C.byref(nb))
        out = np.empty(nb.value, dtype=np.uint8)
        self.lib.ref_archive_fetch(out.ctypes.data, nb.value)
        return out.tobytes()

    def run_pipeline(self, a, dims, blocks, strides, time_chunk, stage1_rank, stage2_tol=1e-6,
                     periodic=None, include_boundary=True, workers=1, qoi="", provenance=""):
        """run_pipeline over the columns of `a` + encode() -> (bytes, stats);
        stats = [fine_entries_peak, coarse_entries_peak, #stage1, #stage2]."""
        a = _f64(a)
        m, n = a.shape
        nax = len(dims)
        if self.lib.ref_run_pipeline.argtypes is None:
            self.lib.ref_run_pipeline.argtypes = [
                _D, _sz, _sz, _SZ, C.POINTER(C.c_int), _sz, _SZ, _SZ, C.c_int, _sz, _sz, C.c_double,
                _sz, C.c_char_p, C.c_char_p, _SZ, _SZ, C.c_char_p, _sz]
        d, p, s, _ = _Port._spec(dims, strides, periodic)
        b = (C.c_size_t * nax)(*blocks)
        nb = C.c_size_t(0)
        stats = (C.c_size_t * 4)()
        err = C.create_string_buffer(512)
        if self.lib.ref_run_pipeline(_dp(a), m, n, d, p, nax, b, s, int(include_boundary), time_chunk,
                                     stage1_rank, stage2_tol, workers, qoi.encode(), provenance.encode(),
                                     C.byref(nb), stats, err, 512):
            name, _, what = err.value.decode().partition("|")
            e = OracleError(name)
            e.what = what
            raise e
        out = np.empty(nb.value, dtype=np.uint8)
        self.lib.ref_archive_fetch(out.ctypes.data, nb.value)
        return out.tobytes(), list(stats)

    def archive_decompress(self, data):
        b = np.frombuffer(bytes(data), dtype=np.uint8)
        m, n = C.c_size_t(0), C.c_size_t(0)
        self._call(self.lib.ref_archive_decompress, b.ctypes.data, b.size, None, 0, C.byref(m),
                   C.byref(n))
        out = np.empty((m.value, n.value), order="F")
        self._call(self.lib.ref_archive_decompress, b.ctypes.data, b.size, _dp(out), out.size,
                   C.byref(m), C.byref(n))
        return out

    def archive_info(self, data):
        b = np.frombuffer(bytes(data), dtype=np.uint8)
        buf = C.create_string_buffer(1 << 20)
        self._call(self.lib.ref_archive_info, b.ctypes.data, b.size, buf, 1 << 20)
        return buf.value.decode()

    def crc32(self, data):
        b = np.frombuffer(bytes(data), dtype=np.uint8)
        return int(self.lib.ref_crc32(b.ctypes.data if b.size else None, b.size))

    def spid(self, a, dims, strides, rank=None, tol=None, periodic=None, include_boundary=True):
        """spid::spid + reconstruct(SpidFactors) (proj/src/id.cpp:62-96): IdResult
        with the COARSE skeleton; .y holds the reconstruction."""
        a = _f64(a)
        m, n = a.shape
        mode, k, t, _ = _rule_args(rank, tol)
        d, p, s, nax = _Port._spec(dims, strides, periodic)
        kcap = max(1, min(m, n))
        mc = m  # upper bound for the coarse rows
        idx = np.zeros(kcap, dtype=np.int64)
        coeffs = np.zeros((kcap, n), order="F")
        skel = np.zeros((mc * kcap,))
        approx = np.zeros((m, n), order="F")
        rk, res = C.c_size_t(0), C.c_double(0)
        self._call(self.lib.ref_spid, _dp(a), m, n, d, p, s, nax, int(include_boundary), mode, k,
                   t, kcap, _ip(idx), _dp(coeffs), _dp(skel), _dp(approx), C.byref(rk),
                   C.byref(res))
        k_ = rk.value
        rows = len(port().row_indices(dims, strides, periodic, include_boundary))
        sk = np.asfortranarray(skel[:rows * k_].reshape(k_, rows).T)
        return IdResult(idx[:k_].copy(), np.asfortranarray(coeffs[:k_]), sk, k_, res.value, approx)

    def interp_apply(self, dims, strides, coarse, periodic=None, include_boundary=True):
        d, p, s, nax = _Port._spec(dims, strides, periodic)
        coarse = _f64(coarse)
        fine = np.zeros((int(np.prod(dims)), coarse.shape[1]), order="F")
        self._call(self.lib.ref_interp_apply, d, p, s, nax, int(include_boundary), _dp(coarse),
                   coarse.shape[1], _dp(fine))
        return fine

    @staticmethod
    def _call(fn, *args):
        err = C.create_string_buffer(128)
        if fn(*args, err, 128):
            raise OracleError(err.value.decode())

    def matmul(self, a, b):
        a, b = _f64(a), _f64(b)
        c = np.empty((a.shape[0], b.shape[1]), order="F")
        self._call(self.lib.ref_matmul, _dp(a), a.shape[0], a.shape[1], _dp(b), b.shape[1], _dp(c))
        return c

    def qr(self, a, rank=None, tol=None, at_most=False):
        a = _f64(a)
        m, n = a.shape
        mode, k, t, _ = _rule_args(rank, tol)
        kcap = max(1, min(m, n))
        q = np.zeros((m, kcap), order="F")
        r = np.zeros((kcap, n), order="F")
        piv = np.zeros(n, dtype=np.int64)
        rk, res = C.c_size_t(0), C.c_double(0)
        self._call(self.lib.ref_qr, _dp(a), m, n, mode, k, t, 1 if at_most else 0, kcap, _dp(q),
                   _dp(r), _ip(piv), C.byref(rk), C.byref(res))
        k_ = rk.value
        return QrResult(np.asfortranarray(q[:, :k_]), np.asfortranarray(r[:k_]), piv, k_,
                        res.value)

    def column_id(self, a, rank=None, tol=None, at_most=False):
        a = _f64(a)
        m, n = a.shape
        mode, k, t, _ = _rule_args(rank, tol)
        kcap = max(1, min(m, n))
        idx = np.zeros(kcap, dtype=np.int64)
        coeffs = np.zeros((kcap, n), order="F")
        skel = np.zeros((m, kcap), order="F")
        rk, res = C.c_size_t(0), C.c_double(0)
        self._call(self.lib.ref_column_id, _dp(a), m, n, mode, k, t, 1 if at_most else 0, kcap,
                   _ip(idx), _dp(coeffs), _dp(skel), C.byref(rk), C.byref(res))
        k_ = rk.value
        return IdResult(idx[:k_].copy(), np.asfortranarray(coeffs[:k_]),
                        np.asfortranarray(skel[:, :k_]), k_, res.value)

    def sub_id(self, a, dims, strides, rank=None, tol=None, periodic=None):
        a = _f64(a)
        m, n = a.shape
        mode, k, t, _ = _rule_args(rank, tol)
        nax = len(dims)
        d = (C.c_size_t * nax)(*dims)
        s = (C.c_size_t * nax)(*strides)
        p = (C.c_int * nax)(*([int(bool(x)) for x in periodic] if periodic else [0] * nax))
        kcap = max(1, min(m, n))
        idx = np.zeros(kcap, dtype=np.int64)
        coeffs = np.zeros((kcap, n), order="F")
        skel = np.zeros((m, kcap), order="F")
        rk, res = C.c_size_t(0), C.c_double(0)
        self._call(self.lib.ref_sub_id, _dp(a), m, n, d, p, s, nax, mode, k, t, kcap, _ip(idx),
                   _dp(coeffs), _dp(skel), C.byref(rk), C.byref(res))
        k_ = rk.value
        return IdResult(idx[:k_].copy(), np.asfortranarray(coeffs[:k_]),
                        np.asfortranarray(skel[:, :k_]), k_, res.value)

    def row_indices(self, dims, strides, periodic=None):
        nax = len(dims)
        d = (C.c_size_t * nax)(*dims)
        s = (C.c_size_t * nax)(*strides)
        p = (C.c_int * nax)(*([int(bool(x)) for x in periodic] if periodic else [0] * nax))
        cap = int(np.prod(dims))
        out = np.zeros(cap, dtype=np.int64)
        cnt = C.c_size_t(0)
        self._call(self.lib.ref_row_indices, d, p, s, nax, _ip(out), cap, C.byref(cnt))
        return out[:cnt.value].copy()

    def rel_frob_error(self, exact, approx):
        exact, approx = _f64(exact), _f64(approx)
        out = C.c_double(0)
        self._call(self.lib.ref_rel_frob_error, _dp(exact), _dp(approx), exact.shape[0],
                   exact.shape[1], C.byref(out))
        return out.value

    def compression_factor(self, m, n, stored):
        out = C.c_double(0)
        self._call(self.lib.ref_compression_factor, m, n, stored, C.byref(out))
        return out.value

    def compress_batch(self, a_batch, omega_batch, k, threads):
        """Time the reference CPU compress over a batch (S, n, m) / (S, m, ell).

        a_batch[s] is A_s stored column-major (so row-major (n, m) memory);
        omega_batch[s] is Omega_s column-major ((m, ell) row-major memory).
        Returns (seconds, ranks)."""
        S, n, m = a_batch.shape
        ell = omega_batch.shape[2]
        a_batch = np.ascontiguousarray(a_batch, dtype=np.float64)
        omega_batch = np.ascontiguousarray(omega_batch, dtype=np.float64)
        ranks = np.zeros(S, dtype=np.uintp)
        secs = C.c_double(0)
        self._call(self.lib.ref_compress_batch, _dp(a_batch), m, n, S, _dp(omega_batch), ell, k,
                   int(threads), ranks.ctypes.data_as(_SZ), C.byref(secs))
        return secs.value, ranks.astype(np.int64)


_port = None
_ref = None


def port() -> _Port:
    global _port
    if _port is None:
        _port = _Port()
    return _port


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> _Ref:
    global _ref
    if _ref is None:
        _ref = _Ref()
    return _ref
