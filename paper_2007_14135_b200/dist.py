"""Multi-GPU driver pieces (SURVEY §8(e) / DESIGN.md §8): frames are independent, so the hot path
shards across ranks with no data-path collective; the only collective is the north-star gather of
the per-frame peak lists.  One process per GPU, torch.distributed (NCCL over NVLink on the B200
box; the same functions run on gloo/CPU tensors in the multi-process tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(total: int, world: int, rank: int) -> range:
    """Contiguous frame range of `rank` when `total` frames are split over `world` ranks
    (strong-scaling split; sizes differ by at most one frame)."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def weak_range(per_rank: int, rank: int) -> range:
    """Frames of `rank` when every rank owns its own batch of `per_rank` frames (weak scaling)."""
    return range(rank * per_rank, (rank + 1) * per_rank)


def pack_peaks(idx: torch.Tensor, val: torch.Tensor, npk: torch.Tensor, info: torch.Tensor,
               out: torch.Tensor | None = None) -> torch.Tensor:
    """(..., B, D) idx int32, val f32, (..., B) npk/info int32 -> (..., B, 2D+2) int32 (val bit-cast)."""
    D = idx.shape[-1]
    if out is None:
        out = torch.empty(idx.shape[:-1] + (2 * D + 2,), dtype=torch.int32, device=idx.device)
    out[..., :D] = idx
    out[..., D:2 * D] = val.view(torch.int32)
    out[..., 2 * D] = npk
    out[..., 2 * D + 1] = info
    return out


def unpack_peaks(packed: torch.Tensor, D: int):
    idx = packed[..., :D]
    val = packed[..., D:2 * D].contiguous().view(torch.float32)
    return idx, val, packed[..., 2 * D], packed[..., 2 * D + 1]


def gather_peaks(packed: torch.Tensor, out: torch.Tensor | None = None, group=None) -> torch.Tensor:
    """all_gather of every rank's packed peak lists -> (world, *packed.shape).  NCCL:
    all_gather_into_tensor on the caller's stream; gloo: list all_gather (CPU tests)."""
    world = dist.get_world_size(group)
    if out is None:
        out = torch.empty((world,) + tuple(packed.shape), dtype=packed.dtype, device=packed.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, packed.contiguous(), group=group)
    else:
        dist.all_gather(list(out.unbind(0)), packed.contiguous(), group=group)
    return out
