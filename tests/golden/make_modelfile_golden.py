"""Generate MBUN / RTEN fixtures with the REFERENCE's own writer.

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src:. NUMBA_CACHE_DIR=/tmp/nb \\
        PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_modelfile_golden.py

Writes (``bitunet`` 0.1.0, ``bitunet.modelfile.write_model / write_tensor``):

* ``tiny_masked.mbun`` — base-16 default (all-masked, neg_one) model at 32x32
  from ``synthesize_bundle(cfg, default_rng(3))``;
* ``tiny_binary_f2.mbun`` — all-binary, stem2_float variant from
  ``default_rng(4)``; ``tiny_masked_zero.mbun`` — all-masked zero-padding
  variant from ``default_rng(5)``;
* ``tensors.npz`` + ``t_*.rten`` — f32 / f64 / i32 arrays and a bit-packed
  tensor, with the arrays they hold;
* ``modelfile_forward.npz`` — the reference ``forward`` of each model on a
  fixed 2x32x32 image (logits, mask), so the GPU path can be checked on the
  model it reads back.
"""

from __future__ import annotations

from dataclasses import replace
from pathlib import Path

import numpy as np

import bitunet as R
from bitunet.graph import scale_config

OUT = Path(__file__).resolve().parent

VARIANTS = {
    "tiny_masked": ({}, 3),
    "tiny_binary_f2": ({"precision": "binary", "stem2_float": True}, 4),
    "tiny_masked_zero": ({"pad_mode": "zero"}, 5),
}


def cfg_of(overrides):
    ov = dict(overrides)
    if ov.get("precision") == "binary":
        ov["precision"] = R.PrecisionMap.all_binary()
    cfg = replace(scale_config(R.UNetConfig(), 4), height=32, width=32)
    return replace(cfg, **ov)


def main():
    fwd = {}
    img = np.random.default_rng(11).random((2, 32, 32, 3))
    for name, (ov, seed) in VARIANTS.items():
        cfg = cfg_of(ov)
        model = R.build(cfg, R.synthesize_bundle(cfg, np.random.default_rng(seed)))
        R.modelfile.write_model(model, OUT / f"{name}.mbun")
        res = R.forward(model, img)
        fwd[f"{name}/logits"] = res.logits
        fwd[f"{name}/mask"] = res.mask
    fwd["image"] = img
    np.savez_compressed(OUT / "modelfile_forward.npz", **fwd)

    rng = np.random.default_rng(12)
    arrays = {
        "f32": rng.normal(size=(2, 3, 5)).astype(np.float32),
        "f64": rng.normal(size=(4, 7)),
        "i32": rng.integers(-2**31, 2**31 - 1, size=(3, 3, 2), dtype=np.int64).astype(np.int32),
    }
    for k, a in arrays.items():
        R.modelfile.write_tensor(OUT / f"t_{k}.rten", a)
    bits = rng.choice((-1, 1), size=(1, 3, 5, 70)).astype(np.int8)
    R.modelfile.write_tensor(OUT / "t_bits.rten", R.pack_tensor(bits))
    np.savez_compressed(OUT / "tensors.npz", bits=bits, **arrays)


if __name__ == "__main__":
    main()
