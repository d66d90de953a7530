"""Multi-process plumbing for one-process-per-GPU runs (torchrun): rank environment,
NCCL unique-id distribution, sequence sharding and max-over-ranks device timing.

torch.distributed only carries the 128-byte NCCL id and scalar timings; every tensor byte
of the USP layer moves through libfastusp.so's own NCCL communicators."""
from __future__ import annotations

import os
from dataclasses import dataclass


@dataclass
class RankEnv:
    rank: int
    world: int
    local_rank: int


def rank_env() -> RankEnv:
    return RankEnv(int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
                   int(os.environ.get("LOCAL_RANK", "0")))


def broadcast_bytes(payload: bytes | None, src: int = 0) -> bytes:
    """Rank `src`'s bytes on every rank (torch.distributed object broadcast)."""
    import torch.distributed as dist
    obj = [payload]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def max_over_ranks(value: float, device=None) -> float:
    """MAX all-reduce of a per-rank scalar (the bench's device time per step)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def shard_rows(s: int, world: int, rank: int) -> slice:
    """split_sequence (protocols.cpp:10-21): rank r holds rows [r*S/N, (r+1)*S/N)."""
    if s % world:
        raise ValueError(f"split_sequence: S={s} not divisible by shard count {world}")
    c = s // world
    return slice(rank * c, (rank + 1) * c)


def mesh_groups(world: int, r: int, rank: int):
    """The (ulysses, ring) groups of `rank` on make_mesh(world, r) (mesh.cpp:34-55)."""
    u = world // r
    ri, ui = rank // u, rank % u
    return [ri * u + j for j in range(u)], [i * u + ui for i in range(r)]
