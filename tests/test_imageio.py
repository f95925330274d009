"""Netpbm I/O (host side) against the reference's own
decodes and encodes (tests/golden/make_image_golden.py)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2601_11660_b200 as mb
from conftest import GOLDEN


@pytest.mark.parametrize("name", ["img_rgb8.ppm", "img_gray16.pgm", "img_rgb7.ppm"])
def test_read_image_matches_reference(name):
    z = np.load(GOLDEN / "images.npz")
    got = mb.read_image(GOLDEN / name)
    ref = z[name.split(".")[0]]
    assert got.dtype == np.float64 and got.shape == ref.shape
    assert np.array_equal(got, ref)


def test_write_mask_and_gray_bytes(tmp_path):
    z = np.load(GOLDEN / "images.npz")
    mb.write_mask(tmp_path / "m.pgm", z["mask_in"])
    mb.write_gray(tmp_path / "g.pgm", z["gray_in"])
    assert (tmp_path / "m.pgm").read_bytes() == z["mask_bytes"].tobytes()
    assert (tmp_path / "g.pgm").read_bytes() == z["gray_bytes"].tobytes()


def test_format_errors(tmp_path):
    p = tmp_path / "x.ppm"
    for blob, match in [(b"P3 1 1 255\n\0\0\0", "magic"), (b"P6 2 2", "truncated header"),
                        (b"P6 2 x 255\n", "decimal"), (b"P6 2 2 0\n", "positive"),
                        (b"P6 2 2 70000\n", "65535"), (b"P6 2 2 255\n\0\0", "raster truncated")]:
        p.write_bytes(blob)
        with pytest.raises(mb.FormatError, match=match):
            mb.read_image(p)
