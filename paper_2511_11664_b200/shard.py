"""Multi-GPU plumbing for batches of independent tensors.

Tensors are independent units, so a batch shards across ranks with no
collective on the data path: each rank codes its contiguous slice on its own
GPU and stream.  The only cross-rank traffic is the benchmark's barrier and
the max-over-ranks reduction of step times (torch.distributed, NCCL on GPUs,
gloo in the CPU tests).
"""

from __future__ import annotations


def partition(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced [start, stop) slice of n_items for `rank` of `world`
    (strong scaling, e.g. config C3: 4096 tensors over 1/2/4/8 GPUs)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def weak_seeds(per_rank: int, rank: int) -> range:
    """Seeds of the tensors rank `rank` codes when per-rank work is fixed (weak scaling)."""
    return range(rank * per_rank, (rank + 1) * per_rank)


def reduce_max(value: float, dist=None, device=None) -> float:
    """Max of a scalar over all ranks (identity without a process group)."""
    if dist is None or not dist.is_available() or not dist.is_initialized():
        return float(value)
    import torch

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(value: float, dist=None, device=None) -> float:
    """Sum of a scalar over all ranks (units processed by the whole job)."""
    if dist is None or not dist.is_available() or not dist.is_initialized():
        return float(value)
    import torch

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
