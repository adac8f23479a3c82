"""Multi-GPU plumbing: cells sharded across ranks, no data-path collective.

One process per GPU (torchrun).  The hot path shards by cell / layer port
(SURVEY.md s8e): units are independent across streams and the only sequential
axis (slot order) stays inside a stream, so each rank owns a contiguous range
of cells and never talks to the others until the end, when one all_reduce of a
small metrics vector reports the job-wide numbers (max time, summed slots).
Works with NCCL (GPUs) and gloo (CPU tests).
"""
from __future__ import annotations

import os


def rank_world():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))


def shard_cells(n_cells: int, rank: int, world: int) -> range:
    """Contiguous cell range of `rank` (sizes differ by at most one)."""
    base, extra = divmod(n_cells, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def cell_seed(base_seed: int, cell: int) -> int:
    """Seed per cell = base + cell id (BASELINE.md input convention)."""
    return base_seed + cell


def reduce_metrics(elapsed_ms: float, units: int, device=None):
    """(max elapsed over ranks, total units over ranks) -- the only collective."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return elapsed_ms, units
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=device)
    n = torch.tensor([units], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(n, op=dist.ReduceOp.SUM)
    return float(t.item()), int(n.item())
