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

__all__ = ["shard_bounds", "pack_masks", "unpack_masks", "gather_frames", "ShardedStream", "StreamRunner"]


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
    the (n_frames, ...) concatenation, other ranks return None. ``dst`` and
    every rank here are group-local (``group_dst``), so any subgroup works.
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
        dist.gather(buf, parts, group=group, group_dst=dst)
        return torch.cat([p[:s] for p, s in zip(parts, sizes)], dim=0)
    dist.gather(buf, None, group=group, group_dst=dst)
    return None


class ShardedStream:
    """Frame-stream sharding and the final gather of bit-packed masks.

    Rank r (group-local) of the group owns the contiguous frames
    ``shard_bounds(n_frames, world, r)``; its results go into ``packed``
    (n_local, ceil(per_frame / 8)) uint8 on ``device`` (one bit per mask
    value, ``numpy.packbits(..., bitorder="little")`` per frame) and
    :meth:`gather` brings every rank's rows to ``dst`` in frame order with
    one ``dist.gather``. Device-agnostic: the B200 path is
    :class:`StreamRunner`; the gloo tests drive this class directly.
    """

    def __init__(self, n_frames: int, per_frame: int, *, dist=None, group=None, device="cpu"):
        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group) if dist is not None else 1
        self.rank = dist.get_rank(group) if dist is not None else 0
        self.n_frames, self.per_frame = n_frames, per_frame
        self.lo, self.hi = shard_bounds(n_frames, self.world, self.rank)
        self.n_local = self.hi - self.lo
        self.packed = torch.zeros((max(self.n_local, 1), (per_frame + 7) // 8), dtype=torch.uint8,
                                  device=device)

    def gather(self, dst: int = 0):
        """Packed masks of the whole stream on ``dst`` (host numpy, frame order), else None."""
        local = self.packed[:self.n_local]
        if self.dist is None:
            return local.cpu().numpy()
        out = gather_frames(local, self.n_frames, self.dist, self.group, dst)
        return None if out is None else out.cpu().numpy()


class StreamRunner(ShardedStream):
    """One rank's part of a frame stream sharded over the GPUs of a node (config 4).

    The rank's frames run through its own :class:`Engine` in batches of
    ``batch``: each batch's 8-bit netpbm samples go host -> device on a copy
    stream, are decoded on the GPU (``decode_raster``, the reference's
    ``sample / maxval``), run through the captured forward and reduced to
    bit-packed masks on the device (``pack_mask_bits``). Two buffer sets
    overlap batch i+1's upload with batch i's compute. :meth:`gather` moves
    every rank's packed masks to ``dst`` and down to host memory: there is
    no other cross-rank traffic; logits stay on the device (SURVEY.md 8(e):
    gathered only on request).
    """

    def __init__(self, model, n_frames: int, *, batch: int = 8, dist=None, group=None,
                 device=None):
        from .runtime import Engine

        engine = Engine(model, batch=batch, device=device)
        cfg = model.config
        super().__init__(n_frames, cfg.height * cfg.width * cfg.out_channels, dist=dist, group=group,
                         device=engine.device)
        self.engine = engine
        self.batch = batch
        self.frame_shape = (cfg.height, cfg.width, cfg.in_channels)
        self._raster = None

    def _slots(self):
        eng = self.engine
        eng._ensure_slots()
        if self._raster is None:
            shape = (self.batch,) + self.frame_shape
            self._raster = [torch.zeros(shape, dtype=torch.uint8, device=eng.device) for _ in range(2)]
        return eng

    def run(self, frames: torch.Tensor, maxval: int = 255):
        """Enqueue this rank's shard: ``frames`` = pinned uint8 (n_local, H, W, C)."""
        from .ops import decode_raster, pack_mask_bits

        if tuple(frames.shape) != (self.n_local,) + self.frame_shape or frames.dtype != torch.uint8:
            raise ValueError(f"rank {self.rank} expects uint8 frames {(self.n_local,) + self.frame_shape}")
        eng = self._slots()
        ev = eng._ev
        for i, b0 in enumerate(range(0, self.n_local, self.batch)):
            s = i & 1
            nb = min(self.batch, self.n_local - b0)
            img, lg, mk, g = eng._slots[s]
            rs = self._raster[s]
            with torch.cuda.stream(eng.h2d):
                if eng._used[s]:
                    eng.h2d.wait_event(ev["comp"][s])  # this slot's previous batch consumed
                rs[:nb].copy_(frames[b0:b0 + nb], non_blocking=True)
                ev["h2d"][s].record(eng.h2d)
            with torch.cuda.stream(eng.stream):
                eng.stream.wait_event(ev["h2d"][s])
                decode_raster(rs, maxval, out=img)
                if g is not None:
                    g.replay()
                else:
                    eng._enqueue(img, lg, mk)
                pack_mask_bits(mk[:nb], out=self.packed[b0:b0 + nb])
                ev["comp"][s].record(eng.stream)
            eng._used[s] = True
        return self.packed[:self.n_local]

    def run_resident(self):
        """The shard's forwards with inputs already in HBM (device throughput)."""
        for _ in range(0, self.n_local, self.batch):
            self.engine.run()

    def gather(self, dst: int = 0):
        self.engine.stream.synchronize()
        return super().gather(dst)
