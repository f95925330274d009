"""Netpbm fixtures decoded / encoded by the REFERENCE (bitunet.imageio).

    PYTHONPATH=/root/reference/pkg/src:. NUMBA_CACHE_DIR=/tmp/nb \\
        PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_image_golden.py

Writes ``img_rgb8.ppm`` (P6, maxval 255, header comments), ``img_gray16.pgm``
(P5, maxval 1000, big-endian 16-bit samples), ``img_rgb7.ppm`` (maxval 7) and
``images.npz`` with the reference's ``read_image`` of each, plus the bytes of
its ``write_mask`` / ``write_gray`` on fixed inputs; ``cli_mask.pgm`` /
``cli_logits.rten``: the reference ``bitunet infer`` of ``tiny_masked.mbun``
on ``img_32.ppm``.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

from bitunet import imageio as RI

OUT = Path(__file__).resolve().parent


def main():
    rng = np.random.default_rng(31)
    rgb = rng.integers(0, 256, size=(24, 40, 3), dtype=np.uint8)
    (OUT / "img_rgb8.ppm").write_bytes(b"P6\n# made for parity tests\n40 24\n# maxval next\n255\n"
                                       + rgb.tobytes())
    g16 = rng.integers(0, 1001, size=(17, 9), dtype=np.uint16)
    (OUT / "img_gray16.pgm").write_bytes(b"P5 9 17 1000\n" + g16.astype(">u2").tobytes())
    r7 = rng.integers(0, 8, size=(5, 6, 3), dtype=np.uint8)
    (OUT / "img_rgb7.ppm").write_bytes(b"P6\t6 5\r\n7\n" + r7.tobytes())
    arrays = {k: RI.read_image(OUT / f"{k}.{ext}") for k, ext in
              (("img_rgb8", "ppm"), ("img_gray16", "pgm"), ("img_rgb7", "ppm"))}
    mask = rng.integers(0, 2, size=(1, 7, 5))
    gray = rng.random((6, 4))
    gray[0, 0], gray[0, 1] = 0.5 / 255, -0.1
    RI.write_mask(OUT / "tmp_mask.pgm", mask)
    RI.write_gray(OUT / "tmp_gray.pgm", gray)
    arrays["mask_in"] = mask
    arrays["gray_in"] = gray
    arrays["mask_bytes"] = np.frombuffer((OUT / "tmp_mask.pgm").read_bytes(), dtype=np.uint8)
    arrays["gray_bytes"] = np.frombuffer((OUT / "tmp_gray.pgm").read_bytes(), dtype=np.uint8)
    (OUT / "tmp_mask.pgm").unlink()
    (OUT / "tmp_gray.pgm").unlink()
    np.savez_compressed(OUT / "images.npz", **arrays)

    # the reference CLI end to end on a reference-written model (cli.py:268-288)
    from bitunet.cli import main as ref_main

    img = rng.integers(0, 256, size=(32, 32, 3), dtype=np.uint8)
    (OUT / "img_32.ppm").write_bytes(b"P6\n32 32\n255\n" + img.tobytes())
    rc = ref_main(["infer", "--model", str(OUT / "tiny_masked.mbun"), "--image", str(OUT / "img_32.ppm"),
                   "--mask-out", str(OUT / "cli_mask.pgm"), "--logits-out", str(OUT / "cli_logits.rten"),
                   "--threads", "1"])
    assert rc == 0, rc


if __name__ == "__main__":
    main()
