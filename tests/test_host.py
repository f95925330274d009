"""Host-side mirror of the reference API and the C-ABI library (CPU only)."""

from __future__ import annotations

import ctypes
import hashlib
import json
import re
from dataclasses import replace

import numpy as np
import pytest

import paper_2601_11660_b200 as mb
from conftest import GOLDEN, ROOT, load_golden, tiny_config
from paper_2601_11660_b200 import _lib
from tests_golden_models import VARIANTS, golden_model, golden_model_256


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def digest(model):
    d = {}
    for l in model.layers:
        if l.threshold is not None:
            d[l.name + ".T"] = sha(l.threshold.thresholds)
            d[l.name + ".codes"] = sha(l.threshold.codes)
        w = l.weights
        if w is None:
            continue
        if hasattr(w, "neg"):
            d[l.name + ".pos"] = sha(w.pos.words)
            d[l.name + ".neg"] = sha(w.neg.words)
        elif hasattr(w, "words"):
            d[l.name + ".plane"] = sha(w.words)
        else:
            d[l.name + ".w"] = sha(np.asarray(w, dtype=np.float64))
    return d


# ------------------------------------------------------------- build parity


@pytest.mark.parametrize("variant", sorted(VARIANTS))
def test_build_matches_reference_build(variant):
    want = json.loads((GOLDEN / "build_digest.json").read_text())
    for extent in (16, 32):
        _, _, model = golden_model(variant, extent)
        assert digest(model) == want[f"{variant}@{extent}"]


@pytest.mark.parametrize("gen,seed", [("synth", 1), ("live", 1), ("live", 2)])
def test_build_matches_reference_build_256(gen, seed):
    want = json.loads((GOLDEN / "build_digest.json").read_text())
    _, _, model, _ = golden_model_256(gen, seed)
    assert digest(model) == want[f"{gen}{seed}@256"]


def test_fuse_bn_sign_matches_reference():
    z = load_golden("bn_fusion.npz")
    ft = mb.fuse_bn_sign(z["gamma"], z["beta"], z["mean"], z["var"], float(z["eps"]), z["bias"])
    assert np.array_equal(ft.codes, z["codes"])
    assert np.array_equal(ft.thresholds, z["thresholds"])


def test_fuse_bn_sign_exact_against_float_predicate(rng):
    # criterion 5 (pkg/tests/test_acceptance.py:264-293): thresholds reproduce
    # the float predicate for every accumulator in [-9216, 9216]
    acc = np.arange(-9216, 9217, dtype=np.int64)
    for _ in range(50):
        c = 8
        g = rng.uniform(-2, 2, c)
        g[0] = 0.0
        b, m = rng.normal(size=c), rng.normal(size=c) * 3000
        v, bias = rng.uniform(0, 1e6, c), rng.normal(size=c)
        ft = mb.fuse_bn_sign(g, b, m, v, 1e-5, bias)
        for j in range(c):
            pred = g[j] * ((acc + bias[j]) - m[j]) / np.sqrt(v[j] + 1e-5) + b[j] >= 0.0
            code, t = ft.codes[j], ft.thresholds[j]
            got = (acc >= t) if code == 0 else (acc <= t) if code == 1 else np.full(acc.shape, code == 3)
            assert np.array_equal(got, pred)


# --------------------------------------------------------------- containers


def test_pack_unpack_round_trip(rng):
    v = rng.choice((-1, 1), size=(2, 3, 4, 200)).astype(np.int8)
    t = mb.pack_tensor(v)
    assert t.words.shape == (2, 3, 4, 4)
    assert np.array_equal(mb.unpack_tensor(t), v)
    t.check_pad_lanes()


def test_conv_weights_round_trip(rng):
    segs = (mb.ChannelSegment(0, 6), mb.ChannelSegment(128, 130))
    w = rng.choice((-1, 0, 1), size=(5, 3, 3, 136)).astype(np.int8)
    planes = mb.pack_conv_weights(w, segs, masked=True)
    spec = mb.ConvSpec(3, 3, 1, 1, 136, 5)
    assert np.array_equal(mb.unpack_conv_weights(planes, spec, segs), w)


def test_plane_validation():
    with pytest.raises(mb.LayoutError):
        mb.BitPlane(65, np.zeros(1, np.uint64))
    with pytest.raises(mb.LayoutError):
        mb.BitPlane(3, np.array([8], np.uint64))
    p = mb.BitPlane(3, np.array([1], np.uint64))
    with pytest.raises(mb.PlaneOverlapError):
        mb.MaskedWeightPlanes(p, p)
    with pytest.raises(mb.ValueAlphabetError):
        mb.pack_tensor(np.zeros((1, 1, 1, 2)))


def test_config_api():
    cfg = mb.UNetConfig()
    assert len(mb.layer_specs(cfg)) == 31
    assert mb.validate(cfg) == []
    assert mb.validate(replace(cfg, height=100)) != []
    binary_zero = replace(cfg, pad_mode="zero", precision=mb.PrecisionMap.all_binary())
    assert mb.validate(binary_zero)
    assert mb.PrecisionMap.from_config_id(0x0F0).config_id() == 0x0F0
    with pytest.raises(mb.UnsupportedConfigError):
        mb.scale_config(cfg, 5)
    segs = mb.input_segments(tiny_config())
    assert segs["up-C1.a"] == (mb.ChannelSegment(0, 96), mb.ChannelSegment(128, 128))


def test_live_bundle_is_deterministic():
    cfg = tiny_config(extent=16)
    a = mb.live_bundle(cfg, np.random.default_rng(3))
    b = mb.live_bundle(cfg, np.random.default_rng(3))
    for k in a.entries:
        assert np.array_equal(a[k].weights, b[k].weights)
        assert np.array_equal(a[k].mean, b[k].mean) if a[k].mean is not None else True


# ------------------------------------------------------------------- C-ABI


def test_library_exports_every_declared_symbol():
    header = (ROOT / "include" / "mbunet.h").read_text()
    declared = set(re.findall(r"\b(mbu_[a-z0-9_]+)\s*\(", header))
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.EXPORTED)


def test_library_reports_errors_without_a_gpu():
    lib = _lib.load()
    assert lib.mbu_version() == 1
    h = ctypes.c_void_p()
    offs = np.array([0], np.int32)
    cnts = np.array([4], np.int32)
    pos = np.zeros(9 * 2, np.uint64)
    st = lib.mbu_conv_create(ctypes.byref(h), 0, 0, 3, 3, 1, 1, 4, 1, 1, 1,
                             offs.ctypes.data, cnts.ctypes.data, pos.ctypes.data, None,
                             None, None)
    assert st == 6  # binary + zero padding -> UnsupportedConfigError
    assert b"zero-pad" in lib.mbu_last_error()
    with pytest.raises(mb.UnsupportedConfigError):
        mb.errors.raise_for_status(st, "x")


def test_product_path_refuses_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    x = mb.pack_tensor(np.ones((1, 2, 2, 4), np.int8))
    w = mb.pack_conv_weights(np.ones((2, 3, 3, 4), np.int8), x.segments, masked=True)
    with pytest.raises(mb.EngineError):
        mb.conv_forward(x, w, mb.ConvSpec(3, 3, 1, 1, 4, 2))


def test_product_never_imports_the_oracle():
    for p in (ROOT / "paper_2601_11660_b200").rglob("*.py"):
        src = p.read_text()
        assert "import oracle" not in src and "from oracle" not in src, p
