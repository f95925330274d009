"""GPU build-time quantization: ``mbu_fuse_bn_sign``
against the reference's own fused thresholds (tests/golden/bn_fusion.npz,
made by the reference), and ``quantize_bundle(..., device=)`` equal to the
host path (itself pinned to the reference's build digests)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2601_11660_b200 as mb
from conftest import load_golden, tiny_config
from paper_2601_11660_b200 import ops, quantizer

pytestmark = pytest.mark.gpu


def test_fuse_bn_sign_gpu_matches_reference(cuda):
    z = load_golden("bn_fusion.npz")
    ft = ops.fuse_bn_sign(z["gamma"], z["beta"], z["mean"], z["var"], float(z["eps"]), z["bias"])
    assert np.array_equal(ft.codes, z["codes"])
    assert np.array_equal(ft.thresholds, z["thresholds"])


def test_fuse_bn_sign_gpu_edge_cases(cuda, rng):
    c = 4096
    g = rng.normal(size=c) * rng.choice([1e-12, 1e-3, 1.0, 1e6], size=c)
    g[::17] = 0.0
    g[::29] = -0.0
    b = rng.normal(size=c) * rng.choice([0.0, 1.0, 1e9], size=c)
    m = rng.normal(size=c) * rng.choice([1.0, 3e3, 5e9], size=c)
    v = rng.uniform(0, 1e6, c)
    v[::13] = 0.0
    bias = rng.normal(size=c) * 100
    host = mb.fuse_bn_sign(g, b, m, v, 1e-5, bias)
    dev = ops.fuse_bn_sign(g, b, m, v, 1e-5, bias)
    assert np.array_equal(dev.codes, host.codes)
    assert np.array_equal(dev.thresholds, host.thresholds)
    host0 = mb.fuse_bn_sign(g, b, m, v, 1e-3)
    dev0 = ops.fuse_bn_sign(g, b, m, v, 1e-3)
    assert np.array_equal(dev0.codes, host0.codes) and np.array_equal(dev0.thresholds, host0.thresholds)
    with pytest.raises(mb.ValueAlphabetError):
        ops.fuse_bn_sign(g, b, m, -v - 1, 1e-5)
    with pytest.raises(mb.ValueAlphabetError):
        ops.fuse_bn_sign(g, b, m, v, 0.0)


def test_quantize_weights_gpu(cuda, rng):
    w = rng.standard_normal((64, 3, 3, 32)).astype(np.float32)
    w.flat[::7] = 0.0
    w.flat[5] = np.nan
    for state in ("masked", "binary"):
        want = quantizer.ternarize_values(w, 0.7) if state == "masked" else quantizer.binarize_values(w)
        got = ops.quantize_weights(w, state, 0.7)
        assert got.dtype == np.int8 and np.array_equal(got, want), state
    tern = rng.integers(-1, 2, size=(8, 3, 3, 8)).astype(np.float32)  # already ternary: passes through
    assert np.array_equal(ops.quantize_weights(tern, "masked", 0.7), tern.astype(np.int8))


def test_quantize_weights_gpu_float64(cuda, rng):
    # float64 weights are compared in float64 (no float32 narrowing): values that
    # underflow or round across delta in float32 keep the host's decision
    w = rng.standard_normal((32, 3, 3, 16))
    w.flat[0], w.flat[1], w.flat[2] = -1e-50, 1e-50, -0.0
    delta = 0.7 * np.abs(w).mean(dtype=np.float64)
    w.flat[3] = np.nextafter(delta, np.inf)   # rounds to float32(delta) or below
    w.flat[4] = np.nextafter(-delta, -np.inf)
    for state in ("masked", "binary"):
        want = quantizer.ternarize_values(w, 0.7) if state == "masked" else quantizer.binarize_values(w)
        got = ops.quantize_weights(w, state, 0.7)
        assert np.array_equal(got, want), state
    assert ops.quantize_weights(w, "binary")[0, 0, 0, 0] == -1  # sign(-1e-50) = -1


@pytest.mark.parametrize("gen,seed", [("synth", 3), ("live", 4)])
def test_quantize_bundle_gpu_equals_host(cuda, gen, seed):
    cfg = tiny_config(extent=32, precision=mb.PrecisionMap.from_config_id(seed * 1237 % 4096))
    rng = np.random.default_rng(seed)
    bundle = (mb.synthesize_bundle(cfg, rng, zero_gamma_rate=0.05) if gen == "synth"
              else mb.live_bundle(cfg, rng))
    host = mb.quantize_bundle(bundle, cfg)
    dev = mb.quantize_bundle(bundle, cfg, device="cuda:0")
    assert host.keys() == dev.keys()
    for name in host:
        h, d = host[name], dev[name]
        assert h.kind == d.kind and np.array_equal(h.weights, d.weights), name
        if h.threshold is not None:
            assert np.array_equal(h.threshold.thresholds, d.threshold.thresholds), name
            assert np.array_equal(h.threshold.codes, d.threshold.codes), name
