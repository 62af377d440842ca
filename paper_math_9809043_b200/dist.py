"""torch.distributed plumbing for the z-slab solver (argument marshalling only).

One process per GPU (torchrun); the NCCL communicator the library uses is bootstrapped
from a unique id that rank 0 creates (mss_nccl_unique_id) and broadcasts over the torch
process group.  Everything numeric happens in libmss.so.
"""
from __future__ import annotations

import os
from typing import Optional, Tuple

import numpy as np
import torch
import torch.distributed as dist


def env_ranks() -> Tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def broadcast_bytes(payload: Optional[bytes], n: int = 128, device=None) -> bytes:
    """Broadcast n bytes from rank 0 over the default process group."""
    dev = device if device is not None else ("cuda" if dist.get_backend() == "nccl" else "cpu")
    t = torch.zeros(n, dtype=torch.uint8, device=dev)
    if dist.get_rank() == 0:
        t.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    dist.broadcast(t, src=0)
    return bytes(t.cpu().numpy().tobytes())


def nccl_id_for_group() -> bytes:
    """Rank 0 creates the library's NCCL unique id; every rank returns the same bytes."""
    from . import mss
    uid = mss.nccl_unique_id() if dist.get_rank() == 0 else None
    return broadcast_bytes(uid, 128)


def slab_arrays(arr: np.ndarray, z_range: Tuple[int, int], ndim: int = 3) -> np.ndarray:
    """The rank's z-slab of a cell field (shape (..., nz, ny, nx)): planes [z0, z1)."""
    z0, z1 = z_range
    return np.ascontiguousarray(arr[..., z0:z1, :, :])


def max_over_ranks(value: float) -> float:
    """max of a float over all ranks (timings are reported as the slowest rank)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float) -> float:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
