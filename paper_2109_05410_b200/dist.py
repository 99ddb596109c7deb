"""Process-group plumbing for the z-partitioned multi-GPU path (torch.distributed).

The halo exchange itself runs inside liboocz.so (NCCL send/recv of compressed
radius-4 halos, csrc/halo.cu).  torch.distributed only launches the ranks,
broadcasts the 128-byte NCCL unique id from rank 0, and reduces timings (the
maximum over ranks).  Works with the nccl backend (device tensors) and with
gloo (CPU tensors, used by the tests).
"""
from __future__ import annotations

import os


def env_ranks() -> tuple[int, int, int]:
    """(rank, world, local_rank) from the torchrun environment (1 process if unset)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def slab(rank: int, world: int, nz: int) -> tuple[int, int]:
    """Planes [z0, z1) of the global grid owned by `rank` (contiguous z-slabs)."""
    if nz % world:
        raise ValueError(f"world ({world}) does not divide nz ({nz})")
    s = nz // world
    return rank * s, (rank + 1) * s


def share_nccl_id(dist, rank: int, make_id, device="cpu") -> bytes:
    """Rank 0 calls make_id() (e.g. oocz_get_nccl_id); every rank gets its 128 bytes."""
    import torch
    t = torch.zeros(128, dtype=torch.uint8, device=device)
    if rank == 0:
        raw = make_id()
        if len(raw) != 128:
            raise ValueError("an NCCL unique id has 128 bytes")
        t.copy_(torch.frombuffer(bytearray(raw), dtype=torch.uint8))
    dist.broadcast(t, 0)
    return bytes(t.cpu().tolist())


def max_over_ranks(dist, x: float, device="cpu") -> float:
    """The job's time is the slowest rank's (device-timed) time."""
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(dist, x: float, device="cpu") -> float:
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
