"""Multi-GPU plumbing (host side): contiguous sharding and the one collective.

* Bessel batches shard contiguously with no data-path collective
  (BASELINE north_star: "Batches are sharded contiguously across the GPUs ...
  with no communication").
* The vMF fit shards its N rows; the only exchange is one all-reduce of the
  d-vector of column sums (plus the row count), over NCCL on GPUs (gloo in the
  CPU tests).  Every rank then runs the same scalar fit.
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


def allreduce_colsum(colsum: torch.Tensor, n_local: int, group=None) -> tuple[torch.Tensor, int]:
    """Sum the per-rank column sums in place and the row counts; returns (colsum, n_total)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return colsum, int(n_local)
    dist.all_reduce(colsum, group=group)
    cnt = torch.tensor([float(n_local)], dtype=torch.float64, device=colsum.device)
    dist.all_reduce(cnt, group=group)
    return colsum, int(round(cnt.item()))
