"""Multi-GPU sharding of the batched imaging path.

Scans are independent, so N ranks (one process per GPU, torchrun) each image
their own block of scans: weak scaling with no data-path collective.  The
only collectives are bookkeeping: the max over ranks of a device time (the
bench's step time) and an optional gather of the per-scan detections to
rank 0.  Works with any torch.distributed backend (NCCL on the GPU box,
gloo for the CPU tests).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def world() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def scan_block(rank: int, world_size: int, scans_per_rank: int) -> range:
    """Seeds (= scan indices) owned by ``rank``: a contiguous block per rank."""
    if not 0 <= rank < world_size or scans_per_rank < 0:
        raise ValueError("bad rank / world size / scans per rank")
    return range(rank * scans_per_rank, (rank + 1) * scans_per_rank)


def split_scans(n_total: int, rank: int, world_size: int) -> range:
    """Strong-scaling split of n_total scans (balanced, contiguous)."""
    base, extra = divmod(n_total, world_size)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def max_over_ranks(value: float, device: torch.device | None = None) -> float:
    """Max of a per-rank scalar (e.g. a CUDA-event step time) over all ranks."""
    _, n = world()
    if n == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or torch.device("cpu"))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device: torch.device | None = None) -> float:
    _, n = world()
    if n == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or torch.device("cpu"))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_detections(seeds: range, cells: np.ndarray) -> np.ndarray | None:
    """Gather (seed, ix, iy) rows from every rank to rank 0, ordered by seed."""
    rank, n = world()
    rows = np.concatenate([np.asarray(list(seeds))[:, None], np.asarray(cells).reshape(len(seeds), -1)], axis=1)
    if n == 1:
        return rows
    parts = [None] * n if rank == 0 else None
    dist.gather_object(rows, parts, dst=0)
    if rank != 0:
        return None
    allrows = np.concatenate(parts)
    return allrows[np.argsort(allrows[:, 0], kind="stable")]
