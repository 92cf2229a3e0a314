"""Parity rules between the GPU path and the CPU oracle.

* Pivots: compare selection sequences. At the first mismatch step s, accept
  only if the oracle's two largest residual norms at step s differ by
  <= 1e-12 * max_init (a tie relative to the INITIAL scale, qr.cpp:47-49);
  after an accepted divergence only error and CF are compared.
* Coefficients: relative (max-norm) agreement within
  tol_C = max(1e-10, 1e3 * eps * kappa_hat), kappa_hat = R(0,0)/R(k-1,k-1)
  (the measured drift for reordered summation); the same test
  also reports the well-conditioned prefix.
* Relative reconstruction error: 1e-3 relative (north_star).
"""
from __future__ import annotations

import numpy as np

EPS = np.finfo(np.float64).eps
NEAR_TIE = 1e-12
ERR_RTOL = 1e-3


def residual_norms(y: np.ndarray, selected: list[int]) -> np.ndarray:
    """Residual 2-norms of every column of y after projecting out the span of
    the `selected` columns (fp64 numpy, for near-tie judgement only)."""
    if not selected:
        return np.linalg.norm(y, axis=0)
    q, _ = np.linalg.qr(y[:, selected])
    r = y - q @ (q.T @ y)
    out = np.linalg.norm(r, axis=0)
    out[selected] = -1.0
    return out


def compare_pivots(y: np.ndarray, piv_gpu, piv_orc):
    """Returns (n_equal_prefix, accepted: bool, gap at divergence or None)."""
    piv_gpu, piv_orc = list(map(int, piv_gpu)), list(map(int, piv_orc))
    k = min(len(piv_gpu), len(piv_orc))
    max_init = float(np.max(np.linalg.norm(y, axis=0)))
    for s in range(k):
        if piv_gpu[s] != piv_orc[s]:
            nr = residual_norms(y, piv_orc[:s])
            top = np.sort(nr)[::-1][:2]
            gap = float(top[0] - top[1]) / max_init
            return s, gap <= NEAR_TIE, gap
    return k, len(piv_gpu) == len(piv_orc), None


def kappa_hat(r_diag: np.ndarray) -> float:
    d = np.abs(np.asarray(r_diag, dtype=np.float64))
    return float(d[0] / d[-1]) if len(d) and d[-1] > 0 else np.inf


def tol_coeffs(r_diag) -> float:
    return max(1e-10, 1e3 * EPS * kappa_hat(r_diag))


def rel_maxdiff(a, b) -> float:
    a, b = np.asarray(a), np.asarray(b)
    scale = max(float(np.max(np.abs(b))), 1e-300)
    return float(np.max(np.abs(a - b))) / scale
