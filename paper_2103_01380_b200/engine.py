"""Batched device engine: the hot path over torch CUDA tensors.

Layout in HBM: a batch of S subdomain matrices
A_s (m x n, column-major, the reference DenseMatrix layout) is one
contiguous torch tensor of shape (S, n, m) -- row-major (S, n, m) memory IS
S column-major m x n matrices back to back, lda = m, strideA = m*n. Outputs
follow the reference factor layout (spid::IdFactors, ArchiveBlock):
  indices (S, kcap) int64, selection order
  coeffs  (S, n, kcap) = S column-major kcap x n matrices, source order
  skel    (S, kcap, m) = S column-major m x kcap skeletons
  rank (S,) int64, residual_fro (S,) float64, status (S,) int32
torch is only the allocator / stream provider; every kernel is in
libspidgpu.so, reached through the C ABI.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from ._native import SpidError
from .configs import SpidConfig
from .spid import RankRule


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


@dataclass
class CompressResult:
    indices: torch.Tensor
    coeffs: torch.Tensor
    rank: torch.Tensor
    residual_fro: torch.Tensor
    status: torch.Tensor
    skel: torch.Tensor | None
    sketch: torch.Tensor | None
    kcap: int
    m: int
    n: int

    def check(self):
        """Raise the first failing subdomain's reference error name."""
        st = self.status.cpu().numpy()
        bad = np.nonzero(st)[0]
        if len(bad):
            raise SpidError(N.status_name(int(st[bad[0]])), f"subdomain {int(bad[0])} failed")

    def stored_entries(self) -> torch.Tensor:
        """Per-subdomain skeleton + coefficient entries: k*(m + n)
        (Archive::stored_entries, proj/src/archive.cpp:180-184)."""
        return self.rank * (self.m + self.n)


class Engine:
    """spidgpu handle bound to one device, with torch-allocated buffers.

    One Engine's calls share the handle's device workspace: issue them on one
    stream at a time (use one Engine per concurrent stream), see
    include/spidgpu.h "Workspaces"."""

    def __init__(self, device: int = 0):
        self.device = device
        self.dev = torch.device("cuda", device)
        self.h = N.Handle(device)

    def launches(self) -> int:
        return self.h.launches()

    def reserve(self, m: int, n: int, batch: int, ell: int, kcap: int) -> None:
        """Pre-size the workspaces (spidgpu_reserve): later calls of these
        sizes allocate nothing."""
        self.h.check(N.lib.spidgpu_reserve(self.h.h, m, n, batch, ell, kcap))

    def stream_status(self, stream=None) -> None:
        """Synchronise and raise the first deferred error of batched calls
        (out-of-range gather indices) -- spidgpu_stream_status."""
        self.h.check(N.lib.spidgpu_stream_status(self.h.h, _stream(stream)))

    # ---- inputs -----------------------------------------------------------------
    def alloc_field(self, cfg: SpidConfig, batch: int) -> torch.Tensor:
        return torch.empty((batch, cfg.n, cfg.m), dtype=torch.float64, device=self.dev)

    def generate(self, cfg: SpidConfig, first: int, batch: int, out: torch.Tensor | None = None,
                 heavy: np.ndarray | None = None, stream=None) -> torch.Tensor:
        A = out if out is not None else self.alloc_field(cfg, batch)
        spec = cfg.field_spec()
        hv = None
        if heavy is not None:
            hv = np.ascontiguousarray(heavy, dtype=np.uint8)
        self.h.check(N.lib.spidgpu_field_generate(self.h.h, C.byref(spec), first, batch,
                                                  C.c_void_p(hv.ctypes.data) if hv is not None else None,
                                                  _p(A), cfg.m, cfg.m * cfg.n, _stream(stream)))
        return A

    # ---- hot path ------------------------------------------------------------------
    def omega(self, seed: int = 0, subdomain_base: int = 0, explicit: torch.Tensor | None = None):
        om = N.Omega()
        if explicit is None:
            om.mode, om.seed, om.subdomain_base = N.OMEGA_PHILOX, seed, subdomain_base
        else:
            # explicit: (S, m, ell) tensor = S column-major ell x m matrices
            S, m, ell = explicit.shape
            om.mode, om.omega, om.ldo, om.stride = N.OMEGA_EXPLICIT, explicit.data_ptr(), ell, ell * m
        return om

    def sketch(self, A: torch.Tensor, ell: int, *, seed=0, subdomain_base=0, omega=None,
               out=None, stream=None) -> torch.Tensor:
        S, n, m = A.shape
        Y = out if out is not None else torch.empty((S, n, ell), dtype=torch.float64, device=self.dev)
        om = self.omega(seed, subdomain_base, omega)
        self.h.check(N.lib.spidgpu_sketch_batched(self.h.h, _p(A), m, n, m, m * n, S, ell,
                                                  C.byref(om), _p(Y), ell, ell * n, _stream(stream)))
        return Y

    def cpqr(self, Y: torch.Tensor, rule: RankRule, *, want_qr=False, stream=None):
        S, n, rows = Y.shape
        kcap = rule.cap(rows, n)
        idx = torch.zeros((S, kcap), dtype=torch.int64, device=self.dev)
        coeffs = torch.zeros((S, n, kcap), dtype=torch.float64, device=self.dev)
        rank = torch.zeros(S, dtype=torch.int64, device=self.dev)
        resid = torch.zeros(S, dtype=torch.float64, device=self.dev)
        status = torch.zeros(S, dtype=torch.int32, device=self.dev)
        piv = R = Q = None
        if want_qr:
            piv = torch.zeros((S, n), dtype=torch.int64, device=self.dev)
            R = torch.zeros((S, n, kcap), dtype=torch.float64, device=self.dev)
            Q = torch.zeros((S, kcap, rows), dtype=torch.float64, device=self.dev)
        self.h.check(N.lib.spidgpu_cpqr_id_batched(
            self.h.h, _p(Y), rows, n, rows, rows * n, S, C.byref(rule.c()), kcap, _p(idx),
            _p(coeffs), kcap * n, _p(rank), _p(resid), _p(status), _p(piv), _p(R), _p(Q),
            _stream(stream)))
        res = CompressResult(idx, coeffs, rank, resid, status, None, Y, kcap, rows, n)
        if want_qr:
            return res, piv, R, Q
        return res

    def compress(self, A: torch.Tensor, ell: int, rule: RankRule, *, seed=0, subdomain_base=0,
                 omega=None, want_skel=True, want_sketch=False, out: CompressResult | None = None,
                 stream=None) -> CompressResult:
        """Sketch -> CPQR/coefficients -> skeleton gather for every subdomain
        of the batch (spidgpu_compress_batched)."""
        S, n, m = A.shape
        kcap = rule.cap(ell, n)
        r = out
        if r is None:
            r = CompressResult(
                torch.zeros((S, kcap), dtype=torch.int64, device=self.dev),
                torch.zeros((S, n, kcap), dtype=torch.float64, device=self.dev),
                torch.zeros(S, dtype=torch.int64, device=self.dev),
                torch.zeros(S, dtype=torch.float64, device=self.dev),
                torch.zeros(S, dtype=torch.int32, device=self.dev),
                torch.empty((S, kcap, m), dtype=torch.float64, device=self.dev) if want_skel else None,
                torch.empty((S, n, ell), dtype=torch.float64, device=self.dev) if want_sketch else None,
                kcap, m, n)
        om = self.omega(seed, subdomain_base, omega)
        self.h.check(N.lib.spidgpu_compress_batched(
            self.h.h, _p(A), m, n, m, m * n, S, ell, C.byref(om), C.byref(rule.c()), kcap,
            _p(r.indices), _p(r.coeffs), _p(r.rank), _p(r.residual_fro), _p(r.status),
            _p(r.skel), _p(r.sketch), _stream(stream)))
        return r

    def verify(self, A: torch.Tensor, r: CompressResult, stream=None):
        """(err2, ref2) per subdomain: ||A_s - skel_s C_s||_F^2 and ||A_s||_F^2."""
        S, n, m = A.shape
        err2 = torch.empty(S, dtype=torch.float64, device=self.dev)
        ref2 = torch.empty(S, dtype=torch.float64, device=self.dev)
        self.h.check(N.lib.spidgpu_verify_batched(
            self.h.h, _p(A), m, n, m, m * n, S, _p(r.skel), m, m * r.kcap, _p(r.coeffs), r.kcap,
            r.kcap * n, _p(r.rank), _p(err2), _p(ref2), _stream(stream)))
        return err2, ref2

    def gather(self, A: torch.Tensor, r: CompressResult, stream=None) -> torch.Tensor:
        S, n, m = A.shape
        skel = torch.empty((S, r.kcap, m), dtype=torch.float64, device=self.dev)
        self.h.check(N.lib.spidgpu_gather_batched(self.h.h, _p(A), m, n, m, m * n, S,
                                                  _p(r.indices), r.kcap, _p(r.rank), _p(skel), m,
                                                  m * r.kcap, _stream(stream)))
        return skel

    # ---- SPID proper: coarse-grid skeleton + multilinear lift ------
    @staticmethod
    def block_spec(cfg: SpidConfig, stride: int) -> N.GridSpec:
        """The subdomain's local grid: a b^3 block of the periodic N^3 grid is
        periodic along an axis only if it covers it (proj/src/blocking.cpp:
        84-92); non-periodic local axes pin their last point (grid.cpp:101)."""
        per = [cfg.block == cfg.grid] * 3
        return N.grid_spec([cfg.block] * 3, [stride] * 3, per, True, cfg.qois)

    @staticmethod
    def coarse_rows(spec: N.GridSpec) -> int:
        cnt = C.c_int64(0)
        rc = N.lib.spidgpu_row_indices(C.byref(spec), None, 0, C.byref(cnt))
        if rc:
            raise SpidError(N.status_name(rc), "bad grid spec")
        return cnt.value

    def gather_coarse(self, A: torch.Tensor, r: CompressResult, spec: N.GridSpec,
                      stream=None) -> torch.Tensor:
        """skel_c_s = A_s(J, I_s): the SPID skeleton kept on the coarse rows."""
        S, n, m = A.shape
        mc = self.coarse_rows(spec)
        skel = torch.zeros((S, r.kcap, mc), dtype=torch.float64, device=self.dev)
        self.h.check(N.lib.spidgpu_gather_coarse_batched(
            self.h.h, _p(A), m, n, m, m * n, S, C.byref(spec), _p(r.indices), r.kcap, _p(r.rank),
            _p(skel), mc, mc * r.kcap, _stream(stream)))
        return skel

    def lift(self, skel_c: torch.Tensor, r: CompressResult, spec: N.GridSpec, m: int,
             stream=None) -> torch.Tensor:
        """M * skel_c per subdomain (InterpOperator::apply, bit-exact)."""
        S, kcap, mc = skel_c.shape
        fine = torch.zeros((S, kcap, m), dtype=torch.float64, device=self.dev)
        self.h.check(N.lib.spidgpu_interp_apply_batched(
            self.h.h, C.byref(spec), _p(skel_c), mc, mc * kcap, kcap, _p(r.rank), S, _p(fine), m,
            m * kcap, _stream(stream)))
        return fine

    def verify_coarse(self, A: torch.Tensor, r: CompressResult, skel_c: torch.Tensor,
                      spec: N.GridSpec, stream=None):
        """(err2, ref2) of the SPID reconstruction M * skel_c * C
        (spid::reconstruct(SpidFactors), proj/src/id.cpp:92-96)."""
        S, n, m = A.shape
        lifted = self.lift(skel_c, r, spec, m, stream)
        saved = r.skel
        r.skel = lifted
        try:
            return self.verify(A, r, stream)
        finally:
            r.skel = saved

    def reconstruct(self, r: CompressResult, stream=None) -> torch.Tensor:
        S = r.rank.shape[0]
        out = torch.empty((S, r.n, r.m), dtype=torch.float64, device=self.dev)
        self.h.check(N.lib.spidgpu_reconstruct_batched(
            self.h.h, _p(r.skel), r.m, r.m, r.m * r.kcap, _p(r.coeffs), r.kcap, r.kcap * r.n,
            _p(r.rank), r.n, S, _p(out), r.m, r.m * r.n, _stream(stream)))
        return out

    # ---- end to end from host buffers ------------------------------------------
    def compress_host(self, a_host: torch.Tensor, ell: int, rule: RankRule, *, seed=0,
                      subdomain_base=0, group=8, want_skel=True, verify=False, out=None):
        """spidgpu_compress_host: host (pinned) A in, host factors out; the
        H2D/D2H copies are inside the call, overlapped with compute. `out`
        may pass preallocated (pinned) host tensors keyed like the result."""
        S, n, m = a_host.shape
        kcap = rule.cap(ell, n)
        if out is None:
            pin = a_host.is_pinned()
            mk = lambda shape, dt: torch.zeros(shape, dtype=dt, pin_memory=pin)  # noqa: E731
            out = {
                "indices": mk((S, kcap), torch.int64),
                "coeffs": mk((S, n, kcap), torch.float64),
                "rank": mk((S,), torch.int64),
                "residual_fro": mk((S,), torch.float64),
                "status": mk((S,), torch.int32),
            }
            if want_skel:
                out["skel"] = mk((S, kcap, m), torch.float64)
            if verify:
                out["err2"] = mk((S,), torch.float64)
                out["ref2"] = mk((S,), torch.float64)
        om = self.omega(seed, subdomain_base)
        g = lambda k: C.c_void_p(out[k].data_ptr()) if k in out else None  # noqa: E731
        self.h.check(N.lib.spidgpu_compress_host(
            self.h.h, C.c_void_p(a_host.data_ptr()), m, n, S, ell, C.byref(om), C.byref(rule.c()),
            kcap, group, g("indices"), g("coeffs"), g("skel"), g("rank"), g("residual_fro"),
            g("status"), g("err2"), g("ref2")))
        return out

    def close(self):
        self.h.close()


def rule_for(cfg: SpidConfig) -> RankRule:
    if cfg.adaptive:
        return RankRule.blocked(cfg.k, cfg.kstep, cfg.tol)
    return RankRule.fixed(cfg.k)
