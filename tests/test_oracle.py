"""Pin the CPU oracle before trusting it (CPU only).

* Known answers restated from the reference's own oracle tests
  (``pkg/tests/test_oracle.py:27-129``).
* The dense oracle and the packed-engine port against golden vectors that
  the reference itself produced (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_cases, load_golden, tiny_config
from oracle import dense
from oracle import engine as port

import paper_2601_11660_b200 as mb


# ---------------------------------------------------------------- known answers


def test_zero_weights_give_zero(rng):
    x = rng.choice((-1, 1), size=(1, 4, 4, 3)).astype(np.int8)
    assert not dense.ref_conv(x, np.zeros((2, 3, 3, 3), np.int8), padding=1).any()


def test_unit_selector_passes_input_through(rng):
    x = rng.choice((-1, 1), size=(1, 5, 5, 4)).astype(np.int8)
    w = np.zeros((4, 1, 1, 4), np.int8)
    for j in range(4):
        w[j, 0, 0, j] = 1
    assert np.array_equal(dense.ref_conv(x, w), x.astype(np.int32))


def test_hand_computed_window():
    x = np.array([[1, -1], [-1, 1]], np.int8).reshape(1, 2, 2, 1)
    w = np.ones((1, 2, 2, 1), np.int8)
    assert dense.ref_conv(x, w).reshape(-1).tolist() == [0]
    padded = dense.ref_conv(x, w, padding=1)
    assert padded.shape == (1, 3, 3, 1)
    assert padded[0, 0, 0, 0] == -3 + 1
    assert dense.ref_conv(x, w, padding=1, pad_value=0)[0, 0, 0, 0] == 1


def test_counts_oob_taps_exactly():
    x = np.ones((1, 3, 3, 1), np.int8)
    w = np.ones((1, 3, 3, 1), np.int8)
    acc = dense.ref_conv(x, w, padding=1, pad_value=0)
    assert (acc[0, 1, 1, 0], acc[0, 0, 0, 0], acc[0, 0, 1, 0]) == (9, 4, 6)


def test_rejects_bad_alphabets():
    with pytest.raises(ValueError):
        dense.ref_conv(np.zeros((1, 2, 2, 1)), np.ones((1, 1, 1, 1)))
    with pytest.raises(ValueError):
        dense.ref_conv(np.ones((1, 2, 2, 1)), np.full((1, 1, 1, 1), 2))
    with pytest.raises(ValueError):
        dense.ref_conv(np.ones((1, 2, 2, 1)), np.ones((1, 1, 1, 2)))


def test_tconv_scatters_single_pixel():
    x = np.ones((1, 1, 1, 1), np.int8)
    w = np.arange(-1, 3, dtype=np.int8).clip(-1, 1).reshape(1, 2, 2, 1)
    assert dense.ref_tconv(x, w, 2).reshape(-1).tolist() == [-1, 0, 1, 1]
    with pytest.raises(ValueError):
        dense.ref_tconv(x, np.ones((1, 2, 2, 1)), 3)


def test_pool_is_max_over_windows():
    x = -np.ones((1, 2, 2, 1), np.int8)
    assert dense.ref_pool(x).reshape(-1).tolist() == [-1]
    x[0, 1, 1, 0] = 1
    assert dense.ref_pool(x).reshape(-1).tolist() == [1]
    with pytest.raises(ValueError):
        dense.ref_pool(np.ones((1, 3, 2, 1), np.int8))


def test_threshold_all_codes():
    acc = np.array([-5, 0, 5]).reshape(1, 1, 3, 1).repeat(4, axis=3)
    out = dense.ref_threshold(acc, np.zeros(4, np.int32), np.array([0, 1, 2, 3]))
    assert out[0, 0, :, 0].tolist() == [-1, 1, 1]
    assert out[0, 0, :, 1].tolist() == [1, 1, -1]
    assert out[0, 0, :, 2].tolist() == [-1, -1, -1]
    assert out[0, 0, :, 3].tolist() == [1, 1, 1]
    with pytest.raises(ValueError):
        dense.ref_threshold(acc, np.zeros(4, np.int32), np.array([9, 9, 9, 9]))


def test_bn_sign_of_zero_is_positive():
    out = dense.ref_bn_sign(np.zeros((1, 1, 1, 1)), [1.0], [0.0], [0.0], [1.0], 1e-5)
    assert out.reshape(-1).tolist() == [1]


def test_float_conv_identity_kernel(rng):
    x = rng.normal(size=(1, 4, 4, 2))
    w = np.zeros((2, 1, 1, 2))
    w[0, 0, 0, 0] = w[1, 0, 0, 1] = 1.0
    assert np.allclose(dense.ref_float_conv(x, w), x)
    assert np.allclose(dense.ref_float_conv(x, w, np.array([1.0, -1.0])), x + [1.0, -1.0])


# ------------------------------------------------------------ golden: layers


def test_dense_oracle_matches_reference_layers():
    z, cases = golden_cases()
    for c in cases:
        k = c["key"]
        if c["op"] == "conv":
            ref = dense.ref_conv(z[f"{k}_x"], z[f"{k}_w"], c["s"], c["p"],
                                 0 if c["pad_mode"] == "zero" else -1)
            assert np.array_equal(ref, z[f"{k}_acc"]), k
        elif c["op"] == "gapconv":
            x = np.concatenate([z[f"{k}_xa"], z[f"{k}_xb"]], axis=-1)
            assert np.array_equal(dense.ref_conv(x, z[f"{k}_w"], 1, 1), z[f"{k}_acc"]), k
        elif c["op"] == "tconv":
            assert np.array_equal(dense.ref_tconv(z[f"{k}_x"], z[f"{k}_w"], c["k"]),
                                  z[f"{k}_acc"]), k
        elif c["op"] == "pool":
            got = mb.pack_tensor(dense.ref_pool(z[f"{k}_x"])).words
            assert np.array_equal(got, z[f"{k}_out"]), k
        elif c["op"] == "threshold":
            got = mb.pack_tensor(dense.ref_threshold(z[f"{k}_acc"], z[f"{k}_t"], z[f"{k}_codes"]))
            assert np.array_equal(got.words, z[f"{k}_out"]), k


def test_engine_port_matches_reference_layers():
    z, cases = golden_cases()
    for c in cases:
        k = c["key"]
        if c["op"] != "conv":
            continue
        x = mb.pack_tensor(z[f"{k}_x"])
        planes = mb.pack_conv_weights(z[f"{k}_w"], x.segments, masked=c["masked"])
        assert np.array_equal((planes.pos if c["masked"] else planes).words, z[f"{k}_pos"]), k
        spec = mb.ConvSpec(c["k"], c["k"], c["s"], c["p"], c["c_in"], c["c_out"],
                           pad_mode=c["pad_mode"])
        got = port.conv_forward(x.words, ((0, c["c_in"]),), planes, spec, threads=2)
        assert np.array_equal(got, z[f"{k}_acc"]), k


# ----------------------------------------------------------- golden: forward


def _unpack_words(words, segments):
    return port.unpack(words, tuple((s.lane_offset, s.count) for s in segments))


@pytest.mark.parametrize("variant", ["all-masked", "all-binary", "tconvs-masked",
                                     "stem2-float", "zero-pad"])
def test_dense_forward_matches_reference_trace(variant):
    from tests_golden_models import golden_model

    z = load_golden("forward_tiny.npz")
    for extent in (16, 32):
        key = f"{variant}@{extent}"
        cfg, bundle, model = golden_model(variant, extent)
        recs = mb.dense_records(mb.quantize_bundle(bundle, cfg), cfg)
        image = z[f"{key}/image"]
        ref = dense.ref_forward(cfg, recs, image)
        assert np.array_equal(ref["mask"], z[f"{key}/mask"]), key
        assert np.allclose(ref["head"]["out"], z[f"{key}/logits"], rtol=1e-9, atol=1e-9)
        segs = mb.input_segments(cfg)
        names = [l.name for l in model.layers]
        for i, name in enumerate(names):
            acc_key = f"{key}/{name}/acc"
            if acc_key in z.files and np.issubdtype(z[acc_key].dtype, np.integer):
                assert np.array_equal(ref[name]["acc"], z[acc_key]), (key, name)
            out_key = f"{key}/{name}/out"
            if z[out_key].dtype == np.uint64:
                nxt = names[i + 1] if i + 1 < len(names) else None
                seg = segs[nxt] if nxt else None
                got = _unpack_words(z[out_key], seg)
                assert np.array_equal(ref[name]["out"], got), (key, name)


def test_engine_port_forward_matches_reference_words():
    from tests_golden_models import golden_model

    z = load_golden("forward_tiny.npz")
    for variant in ("all-masked", "zero-pad", "stem2-float"):
        key = f"{variant}@16"
        cfg, bundle, model = golden_model(variant, 16)
        logits, mask, trace = port.forward(model, z[f"{key}/image"], threads=2, trace=True)
        assert np.array_equal(mask, z[f"{key}/mask"])
        for name, rec in trace.items():
            if name == "mask":
                continue
            out_key = f"{key}/{name}/out"
            if z[out_key].dtype == np.uint64:
                assert np.array_equal(rec["out"], z[out_key]), (key, name)
