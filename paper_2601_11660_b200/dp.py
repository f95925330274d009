"""Data-parallel frame sharding: one process per GPU, no collective on the path.

MBU-Net frames are independent (the batch axis only flattens into the GEMM
M dimension, ``pkg/src/bitunet/layers.py:276``), so a frame stream is split
into contiguous shards, each rank runs its shard through its own resident
:class:`~paper_2601_11660_b200.runtime.Engine`, and the only exchange is a
final gather of the results to rank 0. Masks travel
bit-packed (1 bit per pixel: 256 KB per 1024x2048 frame); logits only on
request.

The helpers take a ``torch.distributed`` process group and work with both
backends: ``nccl`` on the B200 box (tensors on the rank's GPU), ``gloo`` in
the CPU tests (tensors on the host).
"""

from __future__ import annotations

import numpy as np
import torch

__all__ = ["shard_bounds", "pack_masks", "unpack_masks", "gather_frames"]


def shard_bounds(n_frames: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, stop) of ``rank``'s frames; the first ``n % world`` ranks get one more."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    if n_frames < 0:
        raise ValueError("negative frame count")
    base, extra = divmod(n_frames, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def pack_masks(mask: np.ndarray) -> np.ndarray:
    """(n, H, W, C) uint8 {0,1} -> (n, ceil(H*W*C/8)) uint8, little bit order."""
    m = np.ascontiguousarray(mask, dtype=np.uint8).reshape(mask.shape[0], -1)
    return np.packbits(m, axis=1, bitorder="little")


def unpack_masks(packed: np.ndarray, shape) -> np.ndarray:
    n = packed.shape[0]
    per = int(np.prod(shape[1:]))
    bits = np.unpackbits(packed, axis=1, count=per, bitorder="little")
    return bits.reshape((n,) + tuple(shape[1:]))


def gather_frames(local: torch.Tensor, n_frames: int, dist, group=None, dst: int = 0):
    """Gather per-rank frame shards (leading axis) to ``dst``, in frame order.

    ``local`` holds this rank's ``shard_bounds`` frames. Shards are padded to
    the largest shard so a single ``dist.gather`` moves them; ``dst`` returns
    the (n_frames, ...) concatenation, other ranks return None.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = [b - a for a, b in (shard_bounds(n_frames, world, r) for r in range(world))]
    if local.shape[0] != sizes[rank]:
        raise ValueError(f"rank {rank} holds {local.shape[0]} frames, expected {sizes[rank]}")
    cap = max(sizes)
    buf = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]].copy_(local)
    if rank == dst:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.gather(buf, parts, dst=dst, group=group)
        return torch.cat([p[:s] for p, s in zip(parts, sizes)], dim=0)
    dist.gather(buf, None, dst=dst, group=group)
    return None
