"""Multi-GPU plumbing for the LDP batch: image sharding and the histogram
gather.

Images are independent (no cross-image state; the 3x3 halo never crosses an
image), so a batch shards by contiguous image ranges with no collective on
the data path. The only exchange is the final per-image cell-histogram gather
to rank 0. Counts travel as uint16: a cell holds at most cell_rows*cell_cols
pixels (81*91 = 7371 for the 7x6 grid of a 640x490 frame), so the narrowing is
exact whenever cell area < 65536 -- checked, not assumed.
"""
from __future__ import annotations

from typing import List, Optional, Tuple


def shard_range(n_images: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [lo, hi) image range of `rank`; ranges tile [0, n) exactly."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return n_images * rank // world, n_images * (rank + 1) // world


def wire_dtype_ok(max_count: int) -> bool:
    """uint16 on the wire is exact iff every count fits."""
    return 0 <= max_count < 65536


def gather_histograms(hist, dist, rank: int, world: int, wire=None, out: Optional[List] = None):
    """Gather every rank's [images, cells, bins] int32 histogram shard to rank 0.

    hist : this rank's counts (torch int32; CUDA with NCCL, CPU with gloo)
    wire : optional preallocated int16 tensor of hist's shape (reused per step)
    out  : on rank 0, optional list of `world` int16 receive tensors
    Returns, on rank 0, the list of per-rank int16 shards (rank order =
    image order); None elsewhere. Shards must be equally sized (NCCL gather).
    """
    import torch
    if wire is None:
        wire = torch.empty(hist.shape, dtype=torch.int16, device=hist.device)
    wire.copy_(hist)  # exact: counts < 65536 (wire_dtype_ok), int16 bit pattern
    if world == 1 and not (dist.is_available() and dist.is_initialized()):
        return [wire] if rank == 0 else None
    if rank == 0 and out is None:
        out = [torch.empty_like(wire) for _ in range(world)]
    # moved as raw bytes: every backend (NCCL, gloo) carries uint8
    flat = wire.reshape(-1).view(torch.uint8)
    recv = [o.reshape(-1).view(torch.uint8) for o in out] if rank == 0 else None
    dist.gather(flat, recv, dst=0)
    return out if rank == 0 else None


def widen(shards) -> "object":
    """Rank-0 helper: concatenate int16 shards back to exact int64 counts."""
    import torch
    return torch.cat([s.to(torch.int64) & 0xFFFF for s in shards], dim=0)
