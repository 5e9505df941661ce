"""Multi-GPU partitioning of the template-generation path.

The path partitions into independent template DPs — one per profile instance of a batched
sweep (BASELINE cfg5) — so profiles are sharded in contiguous blocks across ranks with no
collective inside the DP; one all-gather of the fixed-size packed template sets
(include/oobleck_plan.h, `oob_dp_run` output layout) assembles the whole set on every rank.
On GPUs the all-gather is the library's own NCCL communicator (oob_nccl_allgather over
NVLink; torch.distributed only bootstraps it); the CPU tests use a gloo process group.  The
bytes gathered are the library's packed output, unchanged.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(num_profiles: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block of profiles owned by `rank`: (first, count).  The first
    num_profiles % world ranks get one extra profile."""
    if world < 1 or not 0 <= rank < world or num_profiles < 0:
        raise ValueError("need world >= 1, 0 <= rank < world, num_profiles >= 0")
    base, extra = divmod(num_profiles, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def allgather_packed(packed: torch.Tensor, per_rank_bytes: int, group=None, comm=None,
                     stream: int = 0) -> torch.Tensor:
    """All-gather every rank's packed template sets (uint8, `per_rank_bytes` each; a rank
    with fewer profiles pads with zeros) into one [world * per_rank_bytes] tensor, rank
    order.  With `comm` (planner.NcclComm, device tensors): one ncclAllGather through the
    library; otherwise the process group's all_gather (gloo, CPU tests)."""
    world = comm.world if comm is not None else dist.get_world_size(group)
    if packed.dtype != torch.uint8 or packed.dim() != 1:
        raise ValueError("packed must be a 1-D uint8 tensor")
    if packed.numel() > per_rank_bytes:
        raise ValueError("packed larger than per_rank_bytes")
    if packed.numel() < per_rank_bytes:
        pad = torch.zeros(per_rank_bytes, dtype=torch.uint8, device=packed.device)
        pad[: packed.numel()] = packed
        packed = pad
    out = torch.empty(world * per_rank_bytes, dtype=torch.uint8, device=packed.device)
    if comm is not None:
        comm.allgather(packed.data_ptr(), out.data_ptr(), per_rank_bytes, stream)
    else:
        dist.all_gather(list(out.view(world, per_rank_bytes).unbind(0)), packed, group=group)
    return out


def unshard(gathered: torch.Tensor, num_profiles: int, world: int, profile_bytes: int) -> torch.Tensor:
    """Drop the per-rank padding: the packed sets of profiles 0..num_profiles-1 in order."""
    per_rank = (num_profiles + world - 1) // world * profile_bytes
    parts = []
    for r in range(world):
        _, cnt = shard(num_profiles, world, r)
        parts.append(gathered[r * per_rank: r * per_rank + cnt * profile_bytes])
    return torch.cat(parts)
