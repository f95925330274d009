"""The GPU stream runner (config 4's per-rank path) on one B200, world size 1:
u8 raster frames -> GPU decode -> CUDA-graph forward -> GPU bit-packed masks
-> gather, against the public forward of the same decoded frames."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2601_11660_b200 as mb
from conftest import tiny_config
from paper_2601_11660_b200 import dp

pytestmark = pytest.mark.gpu


def test_pack_mask_bits_matches_numpy(cuda):
    rng = np.random.default_rng(5)
    for shape in ((3, 16, 16, 1), (2, 5, 7, 3), (1, 1, 9, 1)):
        m = (rng.random(shape) < 0.4).astype(np.uint8)
        got = mb.ops.pack_mask_bits(torch.from_numpy(m).to(cuda)).cpu().numpy()
        assert np.array_equal(got, dp.pack_masks(m)), shape


@pytest.mark.parametrize("n_frames,batch", [(5, 2), (8, 8), (3, 4)])
def test_stream_runner_world1_equals_forward(cuda, n_frames, batch):
    cfg = tiny_config(extent=32)
    model = mb.build(cfg, mb.live_bundle(cfg, np.random.default_rng(9)))
    raster = np.random.default_rng(10).integers(0, 256, (n_frames, 32, 32, 3), dtype=np.uint8)
    runner = dp.StreamRunner(model, n_frames, batch=batch, device=cuda)
    runner.run(torch.from_numpy(raster).pin_memory())
    got = runner.gather()
    images = raster.astype(np.float64) / 255.0
    want = mb.forward(model, images).mask
    assert np.array_equal(dp.unpack_masks(got, want.shape), want)
    assert 0.0 < want.mean() < 1.0
