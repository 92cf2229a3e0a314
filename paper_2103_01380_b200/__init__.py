"""B200-native SPID compression hot path (arXiv 2103.01380).

Drop-in for the reference's per-subdomain compressor (namespace spid in
/root/reference/proj): Gaussian sketch on FP64 tensor cores, batched
column-pivoted QR + coefficient solve, skeleton gather and exact-error
verification, all in libspidgpu.so behind the C ABI in include/spidgpu.h.

    from paper_2103_01380_b200 import spid       # reference-facing API
    from paper_2103_01380_b200.engine import Engine  # batched device API
"""
from ._native import SpidError  # noqa: F401  (fails loudly if the .so is missing)

__all__ = ["SpidError"]
