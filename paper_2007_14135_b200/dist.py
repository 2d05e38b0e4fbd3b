"""Multi-GPU driver pieces (SURVEY §8(e) / DESIGN.md §8): frames are independent, so the hot path
shards across ranks with no data-path collective; the only collective is the north-star gather of
the per-frame peak lists.  One process per GPU, torch.distributed (NCCL over NVLink on the B200
box; the same functions run on gloo/CPU tensors in the multi-process tests).

Strong scaling (BASELINE configs[3]: "65536 frames ... sharded across 1/2/4/8 B200"): a batch of
`total` frames is split into contiguous shards (shard_range), every rank runs the whole hot path
on its shard, and gather_sharded returns the peak lists of all `total` frames, in frame order, on
every rank — bitwise the same lists for any world size, because every frame's result depends only
on that frame (SURVEY §8(e) invariant; tests/test_gpu_sharding.py, tests/test_dist_gloo.py).
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
    elif packed.is_cuda:                       # gloo (tests): stage through host memory
        host = torch.empty(out.shape, dtype=out.dtype)
        dist.all_gather(list(host.unbind(0)), packed.cpu().contiguous(), group=group)
        out.copy_(host)
    else:
        dist.all_gather(list(out.unbind(0)), packed.contiguous(), group=group)
    return out


def shard_sizes(total: int, world: int) -> list:
    return [len(shard_range(total, world, r)) for r in range(world)]


def gather_sharded(packed: torch.Tensor, total: int, out: torch.Tensor | None = None,
                   buf: torch.Tensor | None = None, group=None) -> torch.Tensor:
    """Gather every rank's packed peak lists for its shard_range(total, world, rank) frames
    ((..., B_r, W) int32, the frame axis second to last) into (..., total, W) in frame order on
    every rank.  Shards differ by at most one frame: each rank's block is padded to the largest
    shard for the one all_gather (NCCL all_gather_into_tensor), then the padding is dropped.
    `buf` (world, ..., max_shard, W) and `out` may be preallocated (e.g. for CUDA-graph capture of
    the surrounding step)."""
    world = dist.get_world_size(group)
    sizes = shard_sizes(total, world)
    bmax = max(sizes)
    lead, W = tuple(packed.shape[:-2]), packed.shape[-1]
    if packed.shape[-2] != sizes[dist.get_rank(group)]:
        raise ValueError(f"packed has {packed.shape[-2]} frames, this rank's shard has "
                         f"{sizes[dist.get_rank(group)]}")
    if packed.shape[-2] < bmax:
        pad = torch.zeros(lead + (bmax, W), dtype=packed.dtype, device=packed.device)
        pad[..., :packed.shape[-2], :] = packed
        packed = pad
    if buf is None:
        buf = torch.empty((world,) + lead + (bmax, W), dtype=packed.dtype, device=packed.device)
    gather_peaks(packed, out=buf, group=group)
    if out is None:
        out = torch.empty(lead + (total, W), dtype=packed.dtype, device=packed.device)
    start = 0
    for r, n in enumerate(sizes):
        out[..., start:start + n, :] = buf[r][..., :n, :]
        start += n
    return out
