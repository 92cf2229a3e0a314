"""Multi-GPU plumbing: static subdomain partition + the one scalar reduction.

The path shards naturally: subdomains are independent and no
data moves between GPUs. Each rank generates
and compresses its own range; the only collective is one all-reduce of four
float64 sums [sum err2, sum ref2, sum stored entries, sum raw entries],
from which

  rel_frob_error = sqrt(sum err2 / sum ref2)   (== rel_frob_error of the
      assembled matrix, proj/src/archive.cpp:305-312 -> metrics.cpp:14-21)
  cf = sum raw / sum stored                    (== compression_factor over
      Archive::stored_entries, proj/src/metrics.cpp:5-12, archive.cpp:180-184)

Backend: NCCL on GPUs (32 bytes, latency bound), gloo in the CPU tests.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch
import torch.distributed as dist


def contiguous_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of global subdomain ids for `rank` (configs 3/5)."""
    lo = (rank * total) // world
    hi = ((rank + 1) * total) // world
    return lo, hi


def round_robin(total: int, rank: int, world: int) -> list[int]:
    """Global ids for `rank` dealt round-robin (config 4: spreads the
    spatially clustered heavy subdomains over GPUs)."""
    return list(range(rank, total, world))


@dataclass
class QualityReport:
    """spid::QualityReport (proj/include/spid/metrics.hpp:18-23)."""
    cf: float
    rel_frob_error: float
    stored_entries: int
    raw_entries: int
    block_ranks: list[int] = field(default_factory=list)


def local_sums(err2, ref2, ranks, m: int, n: int) -> torch.Tensor:
    """The 4-vector a rank contributes (float64)."""
    err2 = torch.as_tensor(err2, dtype=torch.float64)
    ref2 = torch.as_tensor(ref2, dtype=torch.float64)
    ranks = torch.as_tensor(ranks, dtype=torch.float64)
    stored = (ranks * float(m + n)).sum()
    raw = float(m) * float(n) * ranks.numel()
    return torch.stack([err2.sum(), ref2.sum(), stored, torch.tensor(raw, dtype=torch.float64)])


def reduce_report(sums: torch.Tensor, group=None, block_ranks=None) -> QualityReport:
    """All-reduce the 4 sums (if a process group is up) and form the report."""
    v = sums.clone()
    if dist.is_available() and dist.is_initialized():
        if dist.get_backend(group) != "nccl":
            v = v.cpu()  # gloo reduces host tensors
        dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)
    e2, r2, stored, raw = (float(x) for x in v.cpu())
    if r2 == 0.0:
        raise ZeroDivisionError("ZeroReference: reference matrix is zero")
    if stored == 0.0:
        raise ZeroDivisionError("ZeroDenominator: stored entry count must be positive")
    return QualityReport(cf=raw / stored, rel_frob_error=math.sqrt(e2 / r2),
                         stored_entries=int(round(stored)), raw_entries=int(round(raw)),
                         block_ranks=list(block_ranks or []))


def gather_ranks(local_ranks: torch.Tensor, group=None) -> list[int]:
    """All-gather per-subdomain ranks (config 4 report); equal-length chunks."""
    if not (dist.is_available() and dist.is_initialized()):
        return [int(x) for x in local_ranks.cpu()]
    world = dist.get_world_size(group)
    bufs = [torch.empty_like(local_ranks) for _ in range(world)]
    dist.all_gather(bufs, local_ranks, group=group)
    return [int(x) for b in bufs for x in b.cpu()]
