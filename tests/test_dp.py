"""Data-parallel sharding and the final gather, world size 2 (and 3) over gloo (CPU).

The B200 path shards frames across ranks with no collective on the data path
(SURVEY.md §8(e)); the only exchange is the result gather to rank 0. These
tests drive the runner's own sharding / gather class (``dp.ShardedStream``,
the base of ``dp.StreamRunner``) with the CPU engine port (oracle/engine.py)
standing in for a rank's GPU forward: the gathered bit-packed masks (and
logits through ``gather_frames``) must equal one process's forward over the
whole stream, frame for frame. ``tests/test_gpu_dp.py`` runs the GPU runner.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_11660_b200 import dp

N_FRAMES = 5


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _stream():
    import paper_2601_11660_b200 as mb
    from conftest import tiny_config

    cfg = tiny_config(extent=16)
    model = mb.build(cfg, mb.live_bundle(cfg, np.random.default_rng(3)))
    frames = np.random.default_rng(4).random((N_FRAMES, 16, 16, 3))
    return model, frames


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import engine

        model, frames = _stream()
        cfg = model.config
        sh = dp.ShardedStream(N_FRAMES, cfg.height * cfg.width * cfg.out_channels, dist=dist)
        a, b = sh.lo, sh.hi
        assert (a, b) == dp.shard_bounds(N_FRAMES, world, rank)
        logits, mask, _ = engine.forward(model, frames[a:b])
        if sh.n_local:
            sh.packed[:sh.n_local] = torch.from_numpy(dp.pack_masks(mask))
        got_mask = sh.gather(dst=0)
        got_logits = dp.gather_frames(torch.from_numpy(logits), N_FRAMES, dist)
        if rank == 0:
            np.savez(out_path, mask=dp.unpack_masks(got_mask, (N_FRAMES,) + mask.shape[1:]),
                     logits=got_logits.numpy())
        else:
            assert got_mask is None and got_logits is None
    finally:
        dist.destroy_process_group()


def test_shard_bounds_cover_stream_in_order():
    for n in (0, 1, 5, 8, 63, 64):
        for world in (1, 2, 3, 4, 8):
            bounds = [dp.shard_bounds(n, world, r) for r in range(world)]
            assert bounds[0][0] == 0 and bounds[-1][1] == n
            assert all(bounds[i][1] == bounds[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in bounds]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        dp.shard_bounds(4, 2, 2)


def test_pack_masks_round_trip(rng):
    m = (rng.random((3, 7, 5, 2)) < 0.5).astype(np.uint8)
    p = dp.pack_masks(m)
    assert p.shape == (3, (7 * 5 * 2 + 7) // 8)
    assert np.array_equal(dp.unpack_masks(p, m.shape), m)


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_shard_and_gather_equals_single_process(tmp_path, world):
    from oracle import engine

    out = tmp_path / "gathered.npz"
    mp.spawn(_worker, args=(world, _free_port(), str(out)), nprocs=world, join=True)
    model, frames = _stream()
    logits, mask, _ = engine.forward(model, frames)
    got = np.load(out)
    assert np.array_equal(got["mask"], mask)
    assert np.array_equal(got["logits"], logits)
    assert 0.0 < mask.mean() < 1.0  # the live generator keeps the mask informative
