"""Process-group plumbing for data parallelism: one process per GPU, torchrun env.

The NCCL communicator that averages gradients is owned by libppo5 (`ppo_comm_init`); torch's
process group only carries its unique id and the max-over-ranks timing reduction."""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env():
    """(rank, world, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def share_bytes(payload: bytes | None, nbytes: int, device) -> bytes:
    """Broadcast `nbytes` bytes from rank 0 (payload ignored on other ranks)."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return payload
    buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)
    if dist.get_rank() == 0:
        buf.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    dist.broadcast(buf, 0)
    return bytes(buf.cpu().tolist())


def max_over_ranks(x: float, device) -> float:
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def make_comm(device):
    """libppo5 NCCL communicator for the current process group (None when world == 1)."""
    from . import _lib as L
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return None
    rank, world = dist.get_rank(), dist.get_world_size()
    uid = L.comm_unique_id() if rank == 0 else None
    uid = share_bytes(uid, L.PPO_COMM_ID_BYTES, device)
    return L.comm_init(uid, rank, world)
