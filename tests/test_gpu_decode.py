"""GPU netpbm decode: ``mbu_decode_raster`` must be
bit-identical to the reference's ``imageio.read_image`` (golden arrays made by
tests/golden/make_image_golden.py), exhaustively over every sample value for
a spread of maxvals, and a forward fed by GPU-decoded rasters must equal the
forward on host-decoded images."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2601_11660_b200 as mb
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["img_rgb8.ppm", "img_gray16.pgm", "img_rgb7.ppm"])
def test_decode_matches_reference_read_image(cuda, name):
    raster, maxval = mb.read_raster(GOLDEN / name)
    ref = np.load(GOLDEN / "images.npz")[name.split(".")[0]]
    got = mb.decode_raster(raster, maxval).cpu().numpy()
    assert got.dtype == np.float64 and got.shape == ref.shape
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("maxval", [1, 3, 7, 10, 100, 254, 255, 256, 257, 1000, 4095, 12345, 65534, 65535])
def test_decode_every_sample_value(cuda, maxval):
    """All sample values 0..maxval (the correctly rounded quotient, no
    reciprocal shortcut can pass this), plus odd counts for the tail path."""
    vals = np.arange(maxval + 1, dtype=np.uint32)
    vals = np.concatenate([vals, vals[::-1][: 1 + maxval % 13]])
    if maxval > 255:
        raster = np.stack([(vals >> 8).astype(np.uint8), (vals & 255).astype(np.uint8)], -1)
        raster = raster.reshape(1, 1, -1, 1, 2)
    else:
        raster = vals.astype(np.uint8).reshape(1, 1, -1, 1)
    got = mb.decode_raster(raster, maxval).cpu().numpy().reshape(-1)
    ref = vals.astype(np.float64) / maxval
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))


def test_decode_errors(cuda):
    with pytest.raises(mb.ShapeError):
        mb.decode_raster(np.zeros((1, 2, 2, 3), np.uint8), 1000)  # 16-bit without byte axis
    with pytest.raises(mb.ShapeError):
        mb.decode_raster(np.zeros((1, 2, 2, 3), np.uint8), 255, out=torch.empty(3, device=cuda, dtype=torch.float64))


@pytest.mark.parametrize("maxval", [255, 1000])
def test_run_stream_raster_equals_host_decode(cuda, maxval):
    cfg = mb.UNetConfig(height=64, width=128)
    rng = np.random.default_rng(5)
    model = mb.build(cfg, mb.live_bundle(cfg, rng))
    eng = mb.Engine(model, batch=2)
    samples = [rng.integers(0, maxval + 1, size=eng.shape, dtype=np.uint32) for _ in range(3)]
    if maxval > 255:
        rasters = [np.stack([(s >> 8).astype(np.uint8), (s & 255).astype(np.uint8)], -1) for s in samples]
    else:
        rasters = [s.astype(np.uint8) for s in samples]
    host_r = [torch.from_numpy(r).pin_memory() for r in rasters]
    logits = [torch.empty(eng.out_shape, dtype=torch.float64).pin_memory() for _ in range(3)]
    masks = [torch.empty(eng.out_shape, dtype=torch.uint8).pin_memory() for _ in range(3)]
    eng.run_stream_raster(host_r, maxval, logits, masks, 5)
    torch.cuda.synchronize()
    for i in (3, 4, 2):  # the last write of each host slot came from step i
        img = samples[i % 3].astype(np.float64) / maxval
        res = mb.runtime.forward(model, img)
        assert np.array_equal(res.mask, masks[i % 3].numpy()), i
        assert np.array_equal(res.logits, logits[i % 3].numpy()), i
