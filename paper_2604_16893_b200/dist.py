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


def gather_records_async(records: torch.Tensor, group=None):
    """As gather_records, but returns (out, work) with the all-gather in flight: on NCCL it runs on the process
    group's own stream once the current stream reaches this point, so the caller can launch K3 behind it and call
    work.wait() (which makes the current stream wait) just before vp_pack_offsets (the H10
    exchange overlaps the resize)."""
    world = dist.get_world_size(group)
    out = torch.empty(world * records.numel(), dtype=records.dtype, device=records.device)
    work = dist.all_gather_into_tensor(out, records.contiguous(), group=group, async_op=True)
    return out, work


def nccl_log_nranks(path_glob: str):
    """Number of ranks NCCL reported at communicator init (NCCL_DEBUG=INFO lines '... nRanks N ...' written to
    NCCL_DEBUG_FILE), or None if no such line was logged."""
    import glob
    import re
    n = None
    for p in glob.glob(path_glob):
        try:
            with open(p, errors="replace") as fh:
                for line in fh:
                    m = re.search(r"nRanks (\d+)", line)
                    if m:
                        n = max(n or 0, int(m.group(1)))
        except OSError:
            pass
    return n
