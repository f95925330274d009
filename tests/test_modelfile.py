"""MBUN / RTEN files against fixtures the reference wrote.

``tests/golden/make_modelfile_golden.py`` produced the files with
``bitunet.modelfile`` itself; here our reader must parse them, our writer must
reproduce them byte for byte, and our ``build`` of the same bundle must
serialize to the same bytes (reference test_acceptance.py:417-439 checks the
same round-trip identity on its side).
"""

from __future__ import annotations

from dataclasses import replace

import numpy as np
import pytest

import paper_2601_11660_b200 as mb
from conftest import GOLDEN

MODELS = {"tiny_masked": ({}, 3), "tiny_binary_f2": ({"precision": "binary", "stem2_float": True}, 4),
          "tiny_masked_zero": ({"pad_mode": "zero"}, 5)}


def cfg_of(overrides):
    ov = dict(overrides)
    if ov.get("precision") == "binary":
        ov["precision"] = mb.PrecisionMap.all_binary()
    return replace(replace(mb.scale_config(mb.UNetConfig(), 4), height=32, width=32), **ov)


@pytest.mark.parametrize("name", sorted(MODELS))
def test_reference_file_round_trips_byte_identical(tmp_path, name):
    src = GOLDEN / f"{name}.mbun"
    model = mb.read_model(src)
    out = tmp_path / "copy.mbun"
    mb.write_model(model, out)
    assert out.read_bytes() == src.read_bytes()


@pytest.mark.parametrize("name", sorted(MODELS))
def test_our_build_serializes_to_the_reference_bytes(tmp_path, name):
    ov, seed = MODELS[name]
    cfg = cfg_of(ov)
    model = mb.build(cfg, mb.synthesize_bundle(cfg, np.random.default_rng(seed)))
    out = tmp_path / "ours.mbun"
    mb.write_model(model, out)
    assert out.read_bytes() == (GOLDEN / f"{name}.mbun").read_bytes()


def test_read_model_content():
    model = mb.read_model(GOLDEN / "tiny_masked.mbun")
    assert model.config == cfg_of({})
    kinds = [l.kind for l in model.layers]
    assert kinds[0] == "float-conv" and kinds[-1] == "float-conv"
    assert kinds.count("maxpool") == 4 and kinds.count("concat") == 4
    for layer in model.layers:
        if layer.kind.startswith("masked-"):
            assert not np.any(layer.weights.pos.words & layer.weights.neg.words)
            assert len(layer.threshold.thresholds) == layer.spec.c_out


@pytest.mark.parametrize("kind", ["f32", "f64", "i32", "bits"])
def test_tensors(tmp_path, kind):
    ref = np.load(GOLDEN / "tensors.npz")
    src = GOLDEN / f"t_{kind}.rten"
    got = mb.read_tensor(src)
    if kind == "bits":
        assert np.array_equal(mb.unpack_tensor(got), ref["bits"])
    else:
        assert got.dtype == ref[kind].dtype and np.array_equal(got, ref[kind])
    out = tmp_path / "t.rten"
    mb.write_tensor(out, got)
    assert out.read_bytes() == src.read_bytes()


def test_format_errors(tmp_path):
    blob = (GOLDEN / "tiny_binary_f2.mbun").read_bytes()
    cases = {
        "bad magic": b"MBUX" + blob[4:],
        "version": blob[:4] + (2).to_bytes(4, "little") + blob[8:],
        "truncated header": blob[:40],
        "truncated payload": blob[: len(blob) // 2],
        "trailing": blob + b"\0",
    }
    for why, data in cases.items():
        p = tmp_path / "bad.mbun"
        p.write_bytes(data)
        with pytest.raises(mb.FormatError, match="byte"):
            mb.read_model(p)
    t = (GOLDEN / "t_f64.rten").read_bytes()
    p = tmp_path / "bad.rten"
    p.write_bytes(t[:-3])
    with pytest.raises(mb.FormatError, match="truncated"):
        mb.read_tensor(p)
    p.write_bytes(t[:8] + bytes([9]) + t[9:])
    with pytest.raises(mb.FormatError, match="dtype"):
        mb.read_tensor(p)
