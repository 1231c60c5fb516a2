"""Frame sharding across GPUs (one process per GPU).

Frames are independent (engine.run_nms takes one DetectionVector, engine.py:296), so a
stream of F frames is split into contiguous shards, one per rank, with no collective on the
data path.  `gather_survivors` is the optional exchange step: it collects every rank's
survivor masks and counts on one rank with torch.distributed (NCCL between GPUs, gloo on
CPU), for callers that need the whole stream's result in one place.
"""

from __future__ import annotations

import torch


def shard_bounds(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, stop) frame range of `rank` out of `world` (balanced to +-1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"invalid rank {rank} of world {world}")
    return total * rank // world, total * (rank + 1) // world


def gather_survivors(keep_mask: torch.Tensor, keep_count: torch.Tensor, total_frames: int, dst: int = 0,
                     group=None):
    """Gather per-rank survivor masks [F_r, W32] int32 and counts [F_r] int32 onto `dst`.

    Returns (masks [total_frames, W32], counts [total_frames]) on `dst`, None elsewhere.
    Shards follow shard_bounds, so rank r's frames land at rows shard_bounds(total, world, r).
    Uses all_gather on zero-padded equal-size blocks (the collective NCCL and gloo share).
    """
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    a, b = shard_bounds(total_frames, world, rank)
    if keep_mask.shape[0] != b - a or keep_count.shape[0] != b - a:
        raise ValueError(f"rank {rank} holds {keep_mask.shape[0]} frames, expected {b - a}")
    per = max(shard_bounds(total_frames, world, r)[1] - shard_bounds(total_frames, world, r)[0] for r in range(world))
    W = keep_mask.shape[1]
    pm = torch.zeros((per, W), dtype=keep_mask.dtype, device=keep_mask.device)
    pm[: b - a] = keep_mask
    pc = torch.zeros((per,), dtype=keep_count.dtype, device=keep_count.device)
    pc[: b - a] = keep_count
    all_m = [torch.empty_like(pm) for _ in range(world)]
    all_c = [torch.empty_like(pc) for _ in range(world)]
    dist.all_gather(all_m, pm, group=group)
    dist.all_gather(all_c, pc, group=group)
    if rank != dst:
        return None
    masks = torch.cat([all_m[r][: shard_bounds(total_frames, world, r)[1] - shard_bounds(total_frames, world, r)[0]]
                       for r in range(world)])
    counts = torch.cat([all_c[r][: shard_bounds(total_frames, world, r)[1] - shard_bounds(total_frames, world, r)[0]]
                        for r in range(world)])
    return masks, counts
