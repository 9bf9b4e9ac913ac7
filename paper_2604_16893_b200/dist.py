"""H10 -- cross-rank packing for clip-sharded batches.

Clips are sharded contiguously over ranks (independent units, no data-path collective).  The only
exchange is one all-gather of every rank's per-clip (t, h, w, tokens) int32 records so that each
rank knows the global token / patch offsets of every clip (micro-batch packing, "dynamic
batching").  The records are produced on the device by vp_plan_records, gathered with
torch.distributed (NCCL over NVLink on GPUs; gloo in the CPU tests) and scanned on the device by
vp_pack_offsets.  pixel_values and position ids never leave their rank.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_clips: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [a, b) of clips for `rank`; blocks differ in size by at most one clip."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad world/rank {world}/{rank}")
    base, extra = divmod(n_clips, world)
    a = rank * base + min(rank, extra)
    return a, a + base + (1 if rank < extra else 0)


def gather_records(records: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather equal-length int32 record tensors ([clips_per_rank * 4]) -> [world * clips_per_rank * 4]."""
    world = dist.get_world_size(group)
    out = torch.empty(world * records.numel(), dtype=records.dtype, device=records.device)
    dist.all_gather_into_tensor(out, records.contiguous(), group=group)
    return out
