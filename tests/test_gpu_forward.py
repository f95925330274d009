"""GPU parity of the whole MBU-Net forward — runs on the B200 box.

* Tiny models (5 precision / pad variants, 16x16 and 32x32): every layer's
  int32 accumulators and packed output words must equal the reference's
  golden trace exactly; logits within 1e-9 (the reference's own float
  tolerance, verify.py:23); masks exact.
* Config 1 (1x3x256x256, default widths): per-layer SHA-256 of the
  reference's accumulators / words, logits and mask, for the reference
  generator and the activation-preserving "live" generator.
* Size-independent properties at full config-3 shape: CUDA-graph replay ==
  eager, batch-split invariance, path invariance (tcgen05 vs popcount).
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest
import torch

import paper_2601_11660_b200 as mb
from conftest import load_golden, tiny_config
from oracle import dense
from paper_2601_11660_b200 import _lib
from tests_golden_models import VARIANTS, golden_model, golden_model_256

pytestmark = pytest.mark.gpu

FLOAT_TOL = 1e-9


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


@pytest.mark.parametrize("variant", sorted(VARIANTS))
@pytest.mark.parametrize("path", [_lib.PATH_AUTO, _lib.PATH_POPCOUNT])
def test_tiny_forward_matches_reference_trace(cuda, variant, path, conv_engine):
    z = load_golden("forward_tiny.npz")
    for extent in (16, 32):
        key = f"{variant}@{extent}"
        cfg, bundle, model = golden_model(variant, extent)
        res = mb.runtime.forward(model, z[f"{key}/image"], trace=True, path=path)
        assert np.array_equal(res.mask, z[f"{key}/mask"]), key
        assert np.allclose(res.logits, z[f"{key}/logits"], rtol=FLOAT_TOL, atol=FLOAT_TOL)
        assert res.trace["head"]["acc"] is res.logits
        for layer in model.layers:
            name = layer.name
            out_key, acc_key = f"{key}/{name}/out", f"{key}/{name}/acc"
            got = res.trace[name]
            want_out = z[out_key]
            if want_out.dtype == np.uint64:
                assert np.array_equal(got["out"].words, want_out), (key, name)
            if acc_key in z.files:
                want = z[acc_key]
                if np.issubdtype(want.dtype, np.integer):
                    assert np.array_equal(got["acc"], want), (key, name)
                else:
                    assert np.allclose(got["acc"], want, rtol=FLOAT_TOL, atol=FLOAT_TOL), (key, name)


@pytest.mark.parametrize("gen,seed", [("synth", 1), ("live", 1), ("live", 2)])
def test_config1_256_matches_reference(cuda, gen, seed):
    z = load_golden("forward_256.npz")
    key = f"{gen}{seed}@256"
    cfg, bundle, model, image = golden_model_256(gen, seed)
    res = mb.forward(model, image, trace=True)
    assert np.allclose(res.logits, z[f"{key}/logits"], rtol=FLOAT_TOL, atol=FLOAT_TOL)
    assert np.array_equal(res.mask, z[f"{key}/mask"])
    for layer in model.layers:
        rec = res.trace[layer.name]
        k_out, k_acc = f"{key}/{layer.name}/out_sha", f"{key}/{layer.name}/acc_sha"
        if k_out in z.files:
            assert sha(rec["out"].words) == bytes(z[k_out]).decode(), layer.name
        if k_acc in z.files:
            assert sha(rec["acc"]) == bytes(z[k_acc]).decode(), layer.name


def test_forward_vs_dense_oracle_live_64(cuda):
    for seed in (3, 4):
        cfg = tiny_config(extent=64, precision=mb.PrecisionMap.from_config_id(seed * 997 % 4096))
        rng = np.random.default_rng(seed)
        bundle = mb.live_bundle(cfg, rng)
        model = mb.build(cfg, bundle)
        image = rng.random((2, 64, 64, 3))
        res = mb.forward(model, image, trace=True)
        ref = dense.ref_forward(cfg, mb.dense_records(mb.quantize_bundle(bundle, cfg), cfg), image)
        assert np.array_equal(res.mask, ref["mask"])
        for name, r in ref.items():
            if name == "mask" or r["acc"] is None:
                continue
            if np.issubdtype(np.asarray(r["acc"]).dtype, np.integer):
                assert np.array_equal(res.trace[name]["acc"], r["acc"]), name


def test_reference_model_objects_are_accepted(cuda):
    # duck typing: only attribute names matter (models from bitunet.build work)
    cfg, bundle, model = golden_model("all-masked", 16)
    import types

    layers = tuple(types.SimpleNamespace(**vars(l)) for l in model.layers)
    alien = types.SimpleNamespace(config=cfg, layers=layers)
    img = np.random.default_rng(0).random((1, 16, 16, 3))
    assert np.array_equal(mb.forward(alien, img).mask, mb.forward(model, img).mask)


def test_shape_errors(cuda):
    cfg, bundle, model = golden_model("all-masked", 16)
    with pytest.raises(mb.ShapeError):
        mb.forward(model, np.zeros((1, 16, 16, 4)))
    with pytest.raises(mb.ShapeError):
        mb.forward(model, np.zeros((16, 16, 3)))


def test_engine_graph_replay_and_batch_split_at_config3_shape(cuda):
    """Full 1024x2048 widths: graph == eager; batch of 2 == two batches of 1."""
    cfg = mb.UNetConfig(height=1024, width=2048)
    rng = np.random.default_rng(11)
    model = mb.build(cfg, mb.live_bundle(cfg, rng))
    img = torch.from_numpy(rng.random((2, 1024, 2048, 3))).to(cuda)
    eng = mb.Engine(model, batch=2)
    eng.image.copy_(img)
    eng.run()
    torch.cuda.synchronize()
    mask2, logits2 = eng.mask.clone(), eng.logits.clone()
    eng1 = mb.Engine(model, batch=1, use_graph=False)
    for i in range(2):
        eng1.image.copy_(img[i:i + 1])
        eng1.run()
        torch.cuda.synchronize()
        assert torch.equal(eng1.mask, mask2[i:i + 1])
        assert torch.equal(eng1.logits, logits2[i:i + 1])
    m = mask2.float().mean().item()
    assert 0.02 < m < 0.98, m  # live generator: a non-trivial mask


def test_path_invariance_at_256(cuda, conv_engine):
    cfg, bundle, model, image = golden_model_256("live", 1)
    a = mb.runtime.forward(model, image, path=_lib.PATH_AUTO)
    b = mb.runtime.forward(model, image, path=_lib.PATH_POPCOUNT)
    assert np.array_equal(a.mask, b.mask)
    assert np.array_equal(a.logits, b.logits)


def test_run_stream_matches_graph_replay(cuda):
    """The pipelined serving loop returns exactly what a single replay does."""
    cfg = mb.UNetConfig(height=128, width=256)
    rng = np.random.default_rng(21)
    model = mb.build(cfg, mb.live_bundle(cfg, rng))
    eng = mb.Engine(model, batch=2)
    imgs = [torch.from_numpy(rng.random(eng.shape)).pin_memory() for _ in range(3)]
    logits = [torch.empty(eng.out_shape, dtype=torch.float64).pin_memory() for _ in range(3)]
    masks = [torch.empty(eng.out_shape, dtype=torch.uint8).pin_memory() for _ in range(3)]
    eng.run_stream(imgs, logits, masks, 3)
    torch.cuda.synchronize()
    for i in range(3):
        eng.image.copy_(imgs[i].to(cuda))
        eng.run()
        torch.cuda.synchronize()
        assert torch.equal(eng.mask.cpu(), masks[i]), i
        assert torch.equal(eng.logits.cpu(), logits[i]), i


def test_fast_endpoints_equal_float64_endpoints_full_width(cuda):
    """Stem (float32 + exact recheck) and byte-table head against the
    all-float64 generic kernels on a full 1024x2048 frame."""
    cfg = mb.UNetConfig(height=1024, width=2048)
    rng = np.random.default_rng(12)
    model = mb.build(cfg, mb.live_bundle(cfg, rng))
    img = rng.random((1, 1024, 2048, 3))
    a = mb.forward(model, img)
    _lib.call("mbu_set_option", 1, 1)
    try:
        b = mb.forward(model, img)
    finally:
        _lib.call("mbu_set_option", 1, 0)
    assert np.array_equal(a.mask, b.mask)
    assert np.allclose(a.logits, b.logits, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("name", ["tiny_masked", "tiny_binary_f2", "tiny_masked_zero"])
def test_forward_of_reference_model_file(cuda, name):
    """A model file written by the reference (bitunet.modelfile.write_model)
    runs on the GPU unchanged: mask exact, logits within 1e-9 of the
    reference's own forward."""
    from conftest import GOLDEN

    z = np.load(GOLDEN / "modelfile_forward.npz")
    model = mb.read_model(GOLDEN / f"{name}.mbun")
    res = mb.forward(model, z["image"], device="cuda:0")
    assert np.array_equal(res.mask, z[f"{name}/mask"])
    assert np.allclose(res.logits, z[f"{name}/logits"], rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("classes", [3, 19])
def test_multiclass_head_and_class_map(cuda, classes):
    """Multi-class head: per-channel logits / masks
    against the dense oracle, and the argmax class map against numpy
    (including a NaN logit, which numpy.argmax picks first)."""
    from dataclasses import replace

    cfg = replace(tiny_config(extent=32), out_channels=classes)
    rng = np.random.default_rng(40 + classes)
    bundle = mb.live_bundle(cfg, rng)
    model = mb.build(cfg, bundle)
    image = rng.random((2, 32, 32, 3))
    res = mb.forward(model, image, device="cuda:0")
    ref = dense.ref_forward(cfg, mb.dense_records(mb.quantize_bundle(bundle, cfg), cfg), image)
    assert res.logits.shape == (2, 32, 32, classes)
    assert np.array_equal(res.mask, ref["mask"])
    assert np.allclose(res.logits, ref["head"]["out"], rtol=1e-9, atol=1e-9)
    lg = res.logits.copy()
    lg[0, 1, 2, classes // 2] = np.nan
    lg[1, 3, 4, :] = 0.25  # ties: first index
    got = mb.argmax_classes(lg, device="cuda:0")
    assert got.dtype == np.uint8 and np.array_equal(got, np.argmax(lg, axis=-1))
    gd = mb.argmax_classes(torch.from_numpy(lg).to(cuda))
    assert gd.is_cuda and np.array_equal(gd.cpu().numpy(), np.argmax(lg, axis=-1))


def test_wide_layers_fp4_cap_and_i8_fallback(cuda):
    """1024- and 1056-channel layers: FP4 bias slabs at the 32 KB cap, and past it
    (kind::i8 fallback); fast (bits only) and trace forwards against the dense oracle."""
    cfg = mb.UNetConfig(height=64, width=64, encoder_channels=(64, 128, 1024, 1056),
                        tconv_channels=(256, 128, 64, 32), decoder_channels=(256, 128, 64, 32))
    rng = np.random.default_rng(17)
    bundle = mb.live_bundle(cfg, rng)
    model = mb.build(cfg, bundle)
    image = rng.random((2, 64, 64, 3))
    fast = mb.forward(model, image)
    traced = mb.forward(model, image, trace=True)
    ref = dense.ref_forward(cfg, mb.dense_records(mb.quantize_bundle(bundle, cfg), cfg), image)
    assert np.array_equal(fast.mask, ref["mask"])
    assert np.array_equal(traced.mask, ref["mask"])
    assert np.array_equal(fast.logits, traced.logits)
    for name in ("down-C3.a", "down-C4.a", "down-C4.b"):
        assert np.array_equal(traced.trace[name]["acc"], ref[name]["acc"]), name


@pytest.mark.parametrize("env", [{"MBU_PAIR": "0"}, {"MBU_SB64": "0", "MBU_SB128": "0"},
                                 {"MBU_NO_BLOCK_COMMIT": "1"}])
def test_config1_256_engine_variants(cuda, env):
    """The engine's tile variants that the default build does not pick (one-CTA
    tiles instead of CTA pairs; double-buffered tiles; single-buffered tiles
    without per-block commits) against the same reference digests, each in a
    fresh process (the switches are read once per process)."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    script = Path(__file__).resolve().parent / "run_golden256.py"
    r = subprocess.run([sys.executable, str(script), "live", "1"], capture_output=True, text=True,
                       timeout=900, env={**os.environ, **env})
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    assert "ok" in r.stdout


@pytest.mark.parametrize("n,h,w", [(2, 1024, 2048), (3, 144, 208)])
def test_fused_head_equals_head_kernel(cuda, n, h, w):
    """The 1x1 head folded into up-C4.b's epilogue (MBU_OPT_FUSED_HEAD = 1)
    against the standalone nibble-table head kernel (the default): same
    arithmetic, so logits and masks are identical bit for bit, through both
    forward() and the CUDA-graph Engine; the fused Engine runs one kernel
    fewer (144x208: ragged 128-column tiles)."""
    cfg = mb.UNetConfig(height=h, width=w)
    rng = np.random.default_rng(5)
    model = mb.build(cfg, mb.live_bundle(cfg, rng))
    img = rng.random((n, h, w, 3))
    plain = mb.forward(model, img)
    eng_p = mb.Engine(model, batch=n)
    _lib.call("mbu_set_option", 4, 1)
    try:
        fused = mb.forward(model, img)
        eng_f = mb.Engine(model, batch=n)
    finally:
        _lib.call("mbu_set_option", 4, 0)
    assert np.array_equal(fused.mask, plain.mask)
    assert np.array_equal(fused.logits.view(np.uint64), plain.logits.view(np.uint64))
    assert eng_f.launches_per_run == eng_p.launches_per_run - 1
    for eng in (eng_f, eng_p):
        eng.image.copy_(torch.from_numpy(img))
        eng.run()
    torch.cuda.synchronize()
    assert torch.equal(eng_f.mask, eng_p.mask)
    assert torch.equal(eng_f.logits, eng_p.logits)
    assert np.array_equal(eng_f.logits.cpu().numpy(), fused.logits)


def test_forward_chunks_large_batches(cuda, monkeypatch):
    """forward() splits a batch whose workspace exceeds its budget into
    consecutive chunks of frames (frames are independent): same logits and
    masks as one launch sequence over the whole batch."""
    cfg = mb.UNetConfig(height=144, width=208)
    rng = np.random.default_rng(9)
    model = mb.build(cfg, mb.live_bundle(cfg, rng))
    img = rng.random((5, 144, 208, 3))
    whole = mb.forward(model, img)
    ws1 = mb.runtime.DeviceModel(model, cuda).plan(1, 144, 208, False)
    monkeypatch.setenv("MBU_FORWARD_WS_BYTES", str(2 * ws1))  # two frames per chunk
    part = mb.forward(model, img)
    assert np.array_equal(whole.mask, part.mask)
    assert np.array_equal(whole.logits, part.logits)
