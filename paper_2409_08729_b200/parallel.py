"""Multi-GPU plumbing (host side): contiguous sharding and the one collective.

* Bessel batches shard contiguously with no data-path collective
  (BASELINE north_star: "Batches are sharded contiguously across the GPUs ...
  with no communication").
* The vMF fit shards its N rows; the only exchange is one all-reduce of the
  d column sums with the row count appended (d + 1 doubles), over NCCL on GPUs
  (gloo in the CPU tests).  Every rank then runs the same scalar fit.
"""
from __future__ import annotations

import torch


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of a contiguous, balanced split of n items over `world` ranks."""
    if world <= 0 or not (0 <= rank < world) or n < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def allreduce_colsum(buf: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the per-rank [column sums..., row count] buffers (d + 1 doubles, the
    with_count layout of b200_vmf_colsum_*) in place with ONE all-reduce."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return buf
    dist.all_reduce(buf, group=group)
    return buf
