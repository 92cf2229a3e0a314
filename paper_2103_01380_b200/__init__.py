"""B200-native SPID compression hot path (arXiv 2103.01380).

Drop-in for the reference's per-subdomain compressor (namespace spid in
/root/reference/proj): Gaussian sketch on FP64 tensor cores, batched
column-pivoted QR + coefficient solve, skeleton gather and exact-error
verification, all in libspidgpu.so behind the C ABI in include/spidgpu.h.

    from paper_2103_01380_b200 import spid       # reference-facing API
    from paper_2103_01380_b200.engine import Engine  # batched device API

The native library is loaded on first use of any submodule that needs it
(_native raises ImportError if it is not built -- there is no CPU fallback).
"""

__all__ = ["SpidError"]


def __getattr__(name):
    if name == "SpidError":
        from ._native import SpidError

        return SpidError
    raise AttributeError(name)
