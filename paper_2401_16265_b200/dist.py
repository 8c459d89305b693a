"""Process-group plumbing around the native engine (one process per GPU).

torch.distributed is used only to move the NCCL unique id and to take the
max over ranks of device timings; every data-path collective is issued by the
native engine (co2_aar_* in libco2b200.so) on its own comm stream.
"""
from __future__ import annotations

import os


def env_rank() -> tuple[int, int, int]:
    """(rank, world, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(n: int, rank: int, world: int, align: int = 8) -> tuple[int, int]:
    """Contiguous shard [start, start+count) of rank out of world for the
    sharded (ghost-consistent, C4) outer state.  Boundaries are multiples of
    `align` elements (8 bf16 = 16 B) so every shard keeps 128-bit vector
    alignment; the last rank takes the remainder."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    if n < 0:
        raise ValueError("negative size")
    per = (n + world - 1) // world
    per = (per + align - 1) // align * align
    start = min(rank * per, n)
    end = min(start + per, n)
    return start, end - start


def broadcast_nccl_id(make_id, rank: int, world: int) -> bytes:
    """Rank 0 creates the 128-byte NCCL unique id; everyone receives it."""
    if world == 1:
        return bytes(128)
    import torch.distributed as dist
    obj = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def max_over_ranks(values, device=None):
    """Element-wise max over ranks of a list of floats (device timings)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()
