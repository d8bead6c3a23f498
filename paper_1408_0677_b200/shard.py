"""Row-band sharding of one MLS frame across the ranks of one node.

SURVEY.md §8e: pixel rows are split into contiguous bands, every rank gets
the same global viewport (it depends only on the positions, field.py:596),
the control block is broadcast once per frame (NCCL over NVLink on the GPU
box; gloo in the CPU tests), and there is no per-pixel exchange.  Because
libmdc aligns its pixel tiles in global index space, the union of the bands
is bit-identical to the single-GPU frame.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def row_band(rank: int, world: int, height: int) -> tuple[int, int]:
    """Contiguous rows [r0, r1) of rank ``rank``; bands differ by <= 1 row."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return rank * height // world, (rank + 1) * height // world


def broadcast_controls(tensors, src: int = 0, group=None) -> None:
    """Broadcast the per-frame control block (in place) from ``src``."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        for t in tensors:
            dist.broadcast(t, src=src, group=group)


def gather_bands(local: torch.Tensor, height: int, dst: int = 0, group=None):
    """Assemble (d, rows_r, W) bands into (d, H, W) on ``dst`` (None elsewhere)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return local
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    d, _, w = local.shape
    rows = [row_band(r, world, height) for r in range(world)]
    maxr = max(r1 - r0 for r0, r1 in rows)
    pad = torch.zeros((d, maxr, w), dtype=local.dtype, device=local.device)
    pad[:, : local.shape[1]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    dist.gather(pad, bufs, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([b[:, : r1 - r0] for b, (r0, r1) in zip(bufs, rows)], dim=1)
