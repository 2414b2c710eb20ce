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


def gather_histograms(hist, dist, rank: int, world: int, wire=None, out: Optional[List] = None,
                      max_count: Optional[int] = None):
    """Gather every rank's [images, cells, bins] histogram shard to rank 0.

    hist : this rank's counts (torch; CUDA with NCCL, CPU with gloo): int16 /
           uint16 as the kernel writes them for the wire (ldp_batch with an
           int16 hist), or int32 counts
    wire : optional preallocated int16 tensor of hist's shape (int32 hist only)
    out  : on rank 0, optional list of `world` receive tensors (wire dtype)
    max_count : the largest count a histogram can hold (cell area); int32
           counts go out as int16 only when it is below 65536 -- checked,
           not assumed. None: the shard's own maximum decides (one sync).
    Returns, on rank 0, the list of per-rank shards (rank order = image
    order; uint16 bit patterns in int16, widen() restores the counts, or
    int32 when the counts do not fit); None elsewhere. Shards must be equally
    sized (NCCL gather).
    """
    import torch
    if hist.dtype in (torch.int16, torch.uint16):
        send = hist
    else:
        fits = wire_dtype_ok(max_count) if max_count is not None else wire_dtype_ok(int(hist.max()) if
                                                                                   hist.numel() else 0)
        if fits:
            if wire is None:
                wire = torch.empty(hist.shape, dtype=torch.int16, device=hist.device)
            wire.copy_(hist)  # exact: counts < 65536, int16 bit pattern
            send = wire
        else:
            send = hist  # counts that can reach 65536 stay int32 on the wire
    if world == 1 and not (dist.is_available() and dist.is_initialized()):
        return [send] if rank == 0 else None
    if rank == 0 and out is None:
        out = [torch.empty_like(send) for _ in range(world)]
    # moved as raw bytes: every backend (NCCL, gloo) carries uint8
    flat = send.reshape(-1).view(torch.uint8)
    recv = [o.reshape(-1).view(torch.uint8) for o in out] if rank == 0 else None
    dist.gather(flat, recv, dst=0)
    return out if rank == 0 else None


def widen(shards) -> "object":
    """Rank-0 helper: concatenate gathered shards back to exact int64 counts
    (int16 shards carry uint16 bit patterns)."""
    import torch
    return torch.cat([s.to(torch.int64) & 0xFFFF if s.dtype in (torch.int16, torch.uint16) else s.to(torch.int64)
                      for s in shards], dim=0)
