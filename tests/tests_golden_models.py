"""Rebuild the models the golden fixtures were generated from (no reference needed).

``synthesize_bundle`` here draws in the reference's order, so the same seed
yields the reference's bundle; ``test_host.py`` pins that against
``build_digest.json``.
"""

from __future__ import annotations

from dataclasses import replace

import numpy as np

import paper_2601_11660_b200 as mb
from conftest import tiny_config

SEEDS = {16: 7, 32: 8}
VARIANTS = {
    "all-masked": {},
    "all-binary": {"precision": mb.PrecisionMap.all_binary()},
    "tconvs-masked": {"precision": mb.PrecisionMap.from_config_id(0x0F0)},
    "stem2-float": {"stem2_float": True},
    "zero-pad": {"pad_mode": "zero"},
}


def golden_model(variant: str, extent: int):
    cfg = tiny_config(extent=extent, **VARIANTS[variant])
    bundle = mb.synthesize_bundle(cfg, np.random.default_rng(SEEDS[extent]))
    return cfg, bundle, mb.build(cfg, bundle)


def golden_model_256(gen: str, seed: int):
    cfg = mb.UNetConfig(height=256, width=256)
    rng = np.random.default_rng(seed)
    bundle = mb.synthesize_bundle(cfg, rng) if gen == "synth" else mb.live_bundle(cfg, rng)
    image = np.random.default_rng(seed + 1000).random((1, 256, 256, 3))
    return cfg, bundle, mb.build(cfg, bundle), image
