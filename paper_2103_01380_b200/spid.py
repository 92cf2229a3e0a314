"""Reference-facing API: the pyspid surface (proj/bindings/pymodule.cpp) and
the per-subdomain spid:: functions, each one a call into the C ABI.

Every numerical result comes from libspidgpu.so on the GPU; this module only
moves numpy arrays (Fortran order, the reference's DenseMatrix layout) across
the boundary and turns status codes into SpidError exactly where the
reference throws spid::Error.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from ._native import SpidError

__all__ = [
    "SpidError", "RankRule", "column_id", "column_id_at_most", "qr", "sub_id", "sketch_id",
    "reconstruct", "rel_frob_error", "compression_factor", "philox_omega", "row_indices",
    "make_block_domains", "IdFactors", "SpidFactors", "spid", "interp_apply", "spid_reconstruct",
]


@dataclass
class IdFactors:
    """spid::IdFactors (proj/include/spid/id.hpp:12-19)."""
    skeleton_indices: np.ndarray  # int64, selection order
    coeffs: np.ndarray            # k x n, Fortran
    skeleton: np.ndarray          # m_s x k, Fortran
    source_cols: int
    achieved_rank: int
    qr_residual_fro: float
    sketch: np.ndarray | None = None

    def as_dict(self):
        """pyspid's factors_dict (proj/bindings/pymodule.cpp:48-55)."""
        return {"indices": list(map(int, self.skeleton_indices)), "coeffs": self.coeffs,
                "skeleton": self.skeleton, "rank": self.achieved_rank,
                "residual_fro": self.qr_residual_fro}


class RankRule:
    """spid::RankRule (proj/include/spid/qr.hpp:12-37) plus the blocked
    adaptive rule of BASELINE config 4. Validation errors match the
    reference (BadRankRule)."""

    def __init__(self, mode, k=0, tol=0.0, kstep=0, at_most=False):
        self.mode, self.k, self.tol, self.kstep, self.at_most = mode, int(k), float(tol), int(kstep), bool(at_most)

    @staticmethod
    def fixed(k):
        if k < 1:
            raise SpidError("BadRankRule", "fixed rank must be >= 1")
        return RankRule(N.RULE_FIXED, k=k)

    @staticmethod
    def tolerance(tol):
        if not (0.0 < tol < 1.0):
            raise SpidError("BadRankRule", "tolerance must lie in (0, 1)")
        return RankRule(N.RULE_TOL, tol=tol)

    @staticmethod
    def blocked(kmax, kstep, tol):
        if kmax < 1 or kstep < 1 or not (0.0 < tol < 1.0):
            raise SpidError("BadRankRule", "blocked rule needs kmax, kstep >= 1 and tol in (0,1)")
        return RankRule(N.RULE_BLOCKED, k=kmax, tol=tol, kstep=kstep)

    def c(self) -> N.RankRule:
        return N.RankRule(self.mode, 1 if self.at_most else 0, self.k, self.kstep, self.tol)

    def cap(self, rows, n):
        mn = min(rows, n)
        if self.mode == N.RULE_TOL:
            return max(1, mn)
        if self.mode == N.RULE_BLOCKED:
            return max(1, min(self.k, mn))
        return max(1, min(self.k, mn) if self.at_most else self.k)


def _rule(rank=None, tol=None, rule=None) -> RankRule:
    if rule is not None:
        return rule
    if (rank is None) == (tol is None):
        raise ValueError("pass exactly one of rank= or tol=")  # pymodule.cpp:37-41
    return RankRule.fixed(rank) if rank is not None else RankRule.tolerance(tol)


def _f64(a):
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    if a.ndim != 2:
        raise ValueError("expected a 2-D array")
    return a


def _ptr(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def _h(device):
    return N.handle(device)


def column_id(a, rank=None, tol=None, *, rule=None, device=0) -> IdFactors:
    """spid::column_id (proj/src/id.cpp:40-45), on the GPU."""
    a = _f64(a)
    m, n = a.shape
    r = _rule(rank, tol, rule)
    kcap = r.cap(m, n)
    idx = np.zeros(kcap, dtype=np.int64)
    coeffs = np.zeros((kcap, n), order="F")
    skel = np.zeros((m, kcap), order="F")
    rk, res = C.c_int64(0), C.c_double(0)
    h = _h(device)
    h.check(N.lib.spidgpu_column_id(h.h, _ptr(a), m, n, C.byref(r.c()), kcap, _ptr(idx),
                                    _ptr(coeffs), _ptr(skel), C.byref(rk), C.byref(res)))
    k = rk.value
    return IdFactors(idx[:k].copy(), np.asfortranarray(coeffs[:k]), np.asfortranarray(skel[:, :k]),
                     n, k, res.value)


def column_id_at_most(a, k, *, device=0) -> IdFactors:
    """spid::column_id_at_most (proj/src/id.cpp:47-52)."""
    if k < 1:
        raise SpidError("BadRankRule", "fixed rank must be >= 1")
    r = RankRule(N.RULE_FIXED, k=k, at_most=True)
    return column_id(a, rule=r, device=device)


def qr(a, rank=None, tol=None, *, at_most=False, device=0):
    """spid::pivoted_mgs_qr / _at_most (proj/src/qr.cpp:18-25): dict with
    q (m x rank), r (rank x n, pivoted order), pivots, rank, residual_fro."""
    a = _f64(a)
    m, n = a.shape
    r = _rule(rank, tol)
    if at_most:
        r = RankRule(N.RULE_FIXED, k=r.k, at_most=True)
    kcap = r.cap(m, n)
    q = np.zeros((m, kcap), order="F")
    rr = np.zeros((kcap, n), order="F")
    piv = np.zeros(n, dtype=np.int64)
    rk, res = C.c_int64(0), C.c_double(0)
    h = _h(device)
    h.check(N.lib.spidgpu_qr(h.h, _ptr(a), m, n, C.byref(r.c()), kcap, _ptr(q), _ptr(rr),
                             _ptr(piv), C.byref(rk), C.byref(res)))
    k = rk.value
    return {"q": np.asfortranarray(q[:, :k]), "r": np.asfortranarray(rr[:k]), "pivots": piv,
            "rank": k, "residual_fro": res.value}


# ---- grid / blocking host logic (index arithmetic, mirrors the reference) ----

def _axis_coarse_indices(dims, strides, periodic, include_boundary):
    """SubsampleSpec::axis_coarse_indices (proj/src/grid.cpp:91-106)."""
    axes = []
    for ax, dim in enumerate(dims):
        idx = list(range(0, dim, strides[ax]))
        if include_boundary and not periodic[ax] and idx[-1] != dim - 1:
            idx.append(dim - 1)
        axes.append(idx)
    return axes


def row_indices(dims, strides, periodic=None, include_boundary=True) -> np.ndarray:
    """SubsampleSpec::row_indices for a strided structured spec
    (proj/src/grid.cpp:62-75, 108-130): flattened coarse rows J, ascending."""
    dims = [int(d) for d in dims]
    if not 1 <= len(dims) <= 3 or any(d < 2 for d in dims):
        raise SpidError("BadGridGeom", "structured grids have 1 to 3 axes of >= 2 points")
    periodic = list(periodic) if periodic else [False] * len(dims)
    if len(periodic) != len(dims):
        raise SpidError("BadGridGeom", "periodic flag count must match axis count")
    if len(strides) != len(dims):
        raise SpidError("BadSubsampleSpec", "stride count must match axis count")
    if any(s < 1 for s in strides):
        raise SpidError("BadSubsampleSpec", "strides must be >= 1")
    axes = _axis_coarse_indices(dims, strides, periodic, include_boundary)
    a0 = np.asarray(axes[0], dtype=np.int64)
    a1 = np.asarray(axes[1], dtype=np.int64) if len(axes) > 1 else np.zeros(1, np.int64)
    a2 = np.asarray(axes[2], dtype=np.int64) if len(axes) > 2 else np.zeros(1, np.int64)
    d0 = dims[0]
    d1 = dims[1] if len(dims) > 1 else 1
    flat = a0[None, None, :] + d0 * a1[None, :, None] + d0 * d1 * a2[:, None, None]
    return flat.reshape(-1)


def make_block_domains(dims, blocks_per_axis):
    """make_block_domains row sets (proj/src/blocking.cpp:31-98): blocks
    ordered axis 0 fastest, rows inside a block axis 0 fastest; the last
    block on an axis absorbs the remainder (:12-27)."""
    dims = [int(d) for d in dims]
    if len(blocks_per_axis) != len(dims):
        raise SpidError("BadGridGeom", "blocks_per_axis arity must match axis count")
    segs = []
    for dim, cnt in zip(dims, blocks_per_axis):
        if cnt < 1 or cnt > dim:
            raise SpidError("BlockTooSmall", "blocks per axis must lie in [1, axis dim]")
        base = dim // cnt
        s, at = [], 0
        for b in range(cnt):
            ln = dim - at if b + 1 == cnt else base
            s.append((at, ln))
            at += ln
        segs.append(s)
    while len(segs) < 3:
        segs.append([(0, 1)])
    d0 = dims[0]
    d1 = dims[1] if len(dims) > 1 else 1
    out = []
    for (s2, l2) in segs[2]:
        for (s1, l1) in segs[1]:
            for (s0, l0) in segs[0]:
                i0 = np.arange(s0, s0 + l0)
                i1 = np.arange(s1, s1 + l1)
                i2 = np.arange(s2, s2 + l2)
                flat = i0[None, None, :] + d0 * i1[None, :, None] + d0 * d1 * i2[:, None, None]
                out.append(flat.reshape(-1).astype(np.int64))
    return out


def sub_id(a, dims=None, strides=None, rank=None, tol=None, periodic=None, *, rows=None,
           rule=None, device=0) -> IdFactors:
    """spid::sub_id (proj/src/id.cpp:54-60) / pyspid.sub_id: sketch B = A(J,:)
    on the GPU, column ID of B, fine-grid skeleton A(:, I)."""
    a = _f64(a)
    m, n = a.shape
    if rows is None:
        J = row_indices(dims, strides, periodic)
        if int(np.prod(dims)) != m:
            raise SpidError("GeometryMismatch", "matrix row count does not match grid point count")
    else:
        J = np.asarray(rows, dtype=np.int64)
    J = np.ascontiguousarray(J, dtype=np.int64)
    r = _rule(rank, tol, rule)
    kcap = r.cap(len(J), n)
    idx = np.zeros(kcap, dtype=np.int64)
    coeffs = np.zeros((kcap, n), order="F")
    skel = np.zeros((m, kcap), order="F")
    rk, res = C.c_int64(0), C.c_double(0)
    h = _h(device)
    h.check(N.lib.spidgpu_sub_id(h.h, _ptr(a), m, n, _ptr(J), len(J), C.byref(r.c()), kcap,
                                 _ptr(idx), _ptr(coeffs), _ptr(skel), C.byref(rk), C.byref(res)))
    k = rk.value
    return IdFactors(idx[:k].copy(), np.asfortranarray(coeffs[:k]), np.asfortranarray(skel[:, :k]),
                     n, k, res.value)


def sketch_id(a, ell, rank=None, tol=None, *, omega=None, seed=0, subdomain=0, rule=None,
              want_sketch=False, device=0) -> IdFactors:
    """Gaussian-sketch SubID of one subdomain (the BASELINE north star):
    Y = Omega A on FP64 tensor cores, column ID of Y, fine skeleton A(:, I).
    omega=None -> in-kernel Philox Omega (seed, subdomain); otherwise the
    given ell x m matrix (oracle mode)."""
    a = _f64(a)
    m, n = a.shape
    r = _rule(rank, tol, rule)
    om = N.Omega()
    keep = None
    if omega is None:
        om.mode, om.seed, om.subdomain_base = N.OMEGA_PHILOX, seed, subdomain
    else:
        keep = _f64(omega)
        if keep.shape != (ell, m):
            raise SpidError("DimensionMismatch", "omega must be ell x m")
        om.mode, om.omega, om.ldo, om.stride = N.OMEGA_EXPLICIT, keep.ctypes.data, ell, ell * m
    kcap = r.cap(ell, n)
    y = np.zeros((ell, n), order="F") if want_sketch else None
    idx = np.zeros(kcap, dtype=np.int64)
    coeffs = np.zeros((kcap, n), order="F")
    skel = np.zeros((m, kcap), order="F")
    rk, res = C.c_int64(0), C.c_double(0)
    h = _h(device)
    h.check(N.lib.spidgpu_sketch_id(h.h, _ptr(a), m, n, ell, C.byref(om), C.byref(r.c()), kcap,
                                    _ptr(y), _ptr(idx), _ptr(coeffs), _ptr(skel), C.byref(rk),
                                    C.byref(res)))
    k = rk.value
    return IdFactors(idx[:k].copy(), np.asfortranarray(coeffs[:k]), np.asfortranarray(skel[:, :k]),
                     n, k, res.value, y)


@dataclass
class SpidFactors:
    """spid::SpidFactors (proj/include/spid/id.hpp:21-24): base factors with the
    skeleton on the coarse rows J, plus the (recipe-stored) lift spec."""
    base: IdFactors
    spec: object  # _native.GridSpec

    def stored_entries(self) -> int:
        """k (m_c + n): the coarse skeleton plus the coefficients
        (proj/src/metrics.hpp:13-16, archive.cpp:180-184)."""
        return self.base.skeleton.size + self.base.coeffs.size


def spid(a, dims, strides, rank=None, tol=None, periodic=None, *, include_boundary=True,
         rule=None, reconstruct_approx=True, device=0):
    """spid::spid (proj/src/id.cpp:62-83) / pyspid.spid: row-subsample sketch
    B = A(J, :), column ID of B, skeleton kept on the coarse grid; returns
    pyspid's dict (indices, coeffs, skeleton (coarse), rank, approx) plus the
    SpidFactors under "factors"."""
    a = _f64(a)
    m, n = a.shape
    spec = N.grid_spec(dims, strides, periodic, include_boundary)
    cnt = C.c_int64(0)
    rc = N.lib.spidgpu_row_indices(C.byref(spec), None, 0, C.byref(cnt))
    if rc:
        raise SpidError(N.status_name(rc), "bad subsample spec")
    mc = cnt.value
    r = _rule(rank, tol, rule)
    kcap = r.cap(mc, n)
    idx = np.zeros(kcap, dtype=np.int64)
    coeffs = np.zeros((kcap, n), order="F")
    skel = np.zeros((mc, kcap), order="F")
    rk, res = C.c_int64(0), C.c_double(0)
    h = _h(device)
    h.check(N.lib.spidgpu_spid(h.h, _ptr(a), m, n, C.byref(spec), C.byref(r.c()), kcap, _ptr(idx),
                               _ptr(coeffs), _ptr(skel), C.byref(rk), C.byref(res)))
    k = rk.value
    f = IdFactors(idx[:k].copy(), np.asfortranarray(coeffs[:k]), np.asfortranarray(skel[:, :k]),
                  n, k, res.value)
    out = f.as_dict()
    out["factors"] = SpidFactors(f, spec)
    if reconstruct_approx:
        out["approx"] = spid_reconstruct(out["factors"], device=device)
    return out


def interp_apply(dims, strides, coarse, periodic=None, *, include_boundary=True, nqoi=1, device=0):
    """InterpOperator::from_spec(spec).apply(coarse) (proj/src/interp.cpp:
    45-100, 168-186) on the GPU: the multilinear lift of coarse columns."""
    c = _f64(coarse)
    spec = N.grid_spec(dims, strides, periodic, include_boundary, nqoi)
    P = int(np.prod(dims)) * nqoi
    fine = np.zeros((P, c.shape[1]), order="F")
    h = _h(device)
    h.check(N.lib.spidgpu_interp_apply(h.h, C.byref(spec), _ptr(c), c.shape[0], c.shape[1], _ptr(fine)))
    return fine


def spid_reconstruct(factors: SpidFactors, *, device=0):
    """spid::reconstruct(SpidFactors) (proj/src/id.cpp:92-96): M * skel_c * C."""
    f = factors.base
    s, c = _f64(f.skeleton), _f64(f.coeffs)
    m = 1
    for ax in range(factors.spec.naxes):
        m *= int(factors.spec.dims[ax])
    m *= int(factors.spec.nqoi)
    out = np.zeros((m, c.shape[1]), order="F")
    h = _h(device)
    h.check(N.lib.spidgpu_spid_reconstruct(h.h, C.byref(factors.spec), _ptr(s), s.shape[0], s.shape[1],
                                           _ptr(c), c.shape[0], c.shape[1], _ptr(out)))
    return out


def reconstruct(skeleton, coeffs=None, *, device=0):
    """spid::reconstruct / pyspid.reconstruct (proj/src/id.cpp:85-90)."""
    if isinstance(skeleton, IdFactors):
        f = skeleton
        skeleton, coeffs = f.skeleton, f.coeffs
    s, c = _f64(skeleton), _f64(coeffs)
    if s.shape[1] != c.shape[0]:
        raise SpidError("DimensionMismatch", "inconsistent factor dimensions")
    m, k = s.shape
    n = c.shape[1]
    out = np.zeros((m, n), order="F")
    h = _h(device)
    h.check(N.lib.spidgpu_reconstruct(h.h, _ptr(s), m, k, _ptr(c), n, _ptr(out)))
    return out


def rel_frob_error(exact, approx, *, device=0) -> float:
    """spid::rel_frob_error (proj/src/metrics.cpp:14-21), on the GPU."""
    e, a = _f64(exact), _f64(approx)
    if e.shape != a.shape:
        raise SpidError("DimensionMismatch", "matrices must have equal shapes")
    out = C.c_double(0)
    h = _h(device)
    h.check(N.lib.spidgpu_rel_frob_error(h.h, _ptr(e), _ptr(a), e.shape[0], e.shape[1],
                                         C.byref(out)))
    return out.value


def compression_factor(m, n, stored_entries) -> float:
    """spid::compression_factor (proj/src/metrics.cpp:5-12)."""
    out = C.c_double(0)
    rc = N.lib.spidgpu_compression_factor(int(m), int(n), int(stored_entries), C.byref(out))
    if rc:
        raise SpidError(N.status_name(rc), "compression factor")
    return out.value


def philox_omega(seed, subdomain, ell, m, *, device=0):
    """The exact Omega_s the in-kernel Philox sketch uses (ell x m), copied to
    the host -- so the CPU oracle can be fed the same bits."""
    import torch

    h = _h(device)
    with torch.cuda.device(device):
        buf = torch.empty((m, ell), dtype=torch.float64, device=f"cuda:{device}")
        h.check(N.lib.spidgpu_philox_omega(h.h, seed, subdomain, ell, m, C.c_void_p(buf.data_ptr()),
                                           ell, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return np.asfortranarray(buf.cpu().numpy().T)
