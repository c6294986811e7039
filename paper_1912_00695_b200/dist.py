"""z-slab decomposition across processes (one process per GPU).

The reference has no distributed path (only the emitted text ``ops_partition("")``,
src/opsgen.cpp:561).  Here the grid is split along reference dim 0 ("x", the slowest
axis; the north star's "z-slabs"): rank r owns planes [lo_r, hi_r) plus SO/2 ghost planes
per neighbour for u.  The halo exchange is not a separate collective: each rank's stencil
kernel stores its boundary planes straight into the neighbours' ghost planes through
CUDA-IPC-mapped peer memory (NVLink on a B200 node), then publishes a per-step counter
into the neighbour's memory; the neighbour's next step waits on it.  torch.distributed is
only plumbing here: it moves the <=256-byte IPC descriptors and reduces the per-step
statistics on the host.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np


def slab_bounds(n0: int, world: int, rank: int) -> Tuple[int, int]:
    """Balanced contiguous split of [0, n0) into `world` slabs."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    lo = n0 * rank // world
    hi = n0 * (rank + 1) // world
    return lo, hi


def all_slabs(n0: int, world: int) -> List[Tuple[int, int]]:
    return [slab_bounds(n0, world, r) for r in range(world)]


def check_slabs(n0: int, world: int, halo: int) -> None:
    """Every slab must be at least SO/2 planes thick (its boundary planes feed exactly one
    neighbour's ghosts)."""
    for lo, hi in all_slabs(n0, world):
        if hi - lo < halo:
            raise ValueError(f"slab [{lo},{hi}) thinner than the halo ({halo} planes)")


def exchange_and_link(op, rank: int, world: int, group=None) -> None:
    """Exchange IPC descriptors with the two neighbours and link the halo exchange.
    `op` is a paper_1912_00695_b200.Operator built with slab=slab_bounds(...)."""
    import torch.distributed as dist

    blob = op.export_ghosts()
    blobs: List[Optional[bytes]] = [None] * world
    dist.all_gather_object(blobs, blob, group=group)
    lower = blobs[rank - 1] if rank > 0 else None
    upper = blobs[rank + 1] if rank < world - 1 else None
    op.link_neighbours(lower, upper)
    dist.barrier(group=group)


def reduce_step_max(local: np.ndarray, group=None) -> np.ndarray:
    """Whole-grid max|u| per step = max over ranks (NaN if any rank saw a non-finite cell)."""
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(np.where(np.isnan(local), np.inf, local).astype(np.float64))
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    out = t.numpy().astype(np.float32)
    out[np.isinf(out)] = np.nan
    return out


def reduce_traces(local: np.ndarray, group=None) -> np.ndarray:
    """Receiver traces: each receiver is owned by exactly one rank, the others report 0."""
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(np.ascontiguousarray(local, np.float64))
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.numpy().astype(np.float32)


def gather_level(local_full: np.ndarray, slab: Tuple[int, int], group=None) -> np.ndarray:
    """Assemble a grid-sized level from every rank's owned planes."""
    import torch
    import torch.distributed as dist

    lo, hi = slab
    part = np.zeros_like(local_full)
    part[lo:hi] = local_full[lo:hi]
    t = torch.from_numpy(part.astype(np.float64))
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.numpy().astype(np.float32)
