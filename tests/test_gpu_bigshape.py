"""Parity at the BENCHMARKED shapes against the reference itself (B200 box).

The fixtures are ``bitunet.graph.forward`` (graph.py:413-458) run in the
build container on full frames (``tests/golden/make_golden_big.py``):

* config 3 — bench.py's frames 0 and 7 (``bench_frame``) at 1024x2048 through
  the bench model (``live_bundle`` seed 0) and the reference generator
  (``synthesize_bundle`` seed 0). The GPU runs all eight frames of the bench
  batch at once, so the golden frames sit at batch positions 0 and 7.
* config 5 — one 2160x3840 frame (down-C4 runs at 135x240, so tile
  remainders on both axes are exercised).

Every layer's int32 accumulators and packed output words must hash to the
reference's SHA-256 (traced forward), the mask must be exact and the logits
within the reference's own 1e-9 (verify.py:23) — for the traced forward and
for the CUDA-graph Engine the benchmark times.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest
import torch

import paper_2601_11660_b200 as mb
from conftest import load_golden
from paper_2601_11660_b200 import _lib
from paper_2601_11660_b200.quantizer import bench_frame
from paper_2601_11660_b200.runtime import DeviceModel

pytestmark = pytest.mark.gpu

FLOAT_TOL = 1e-9
LOGIT_STRIDE = 997


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def _text(z, key):
    return bytes(z[key]).decode()


def _model(gen, h, w):
    cfg = mb.UNetConfig(height=h, width=w)
    rng = np.random.default_rng(0)
    bundle = mb.live_bundle(cfg, rng) if gen == "live0" else mb.synthesize_bundle(cfg, rng)
    return mb.build(cfg, bundle)


def _check_outputs(z, key, logits_f, mask_f):
    """logits_f / mask_f: one frame's (H, W, 1) float64 / uint8 host arrays."""
    assert np.array_equal(np.packbits(mask_f.reshape(-1)), z[f"{key}/mask"]), key
    lg = logits_f.reshape(-1)
    np.testing.assert_allclose(lg[::LOGIT_STRIDE], z[f"{key}/logits_sample"], rtol=FLOAT_TOL, atol=FLOAT_TOL)
    st = z[f"{key}/logits_stats"]
    np.testing.assert_allclose([lg.sum(), np.abs(lg).sum(), lg.min(), lg.max()], st,
                               rtol=FLOAT_TOL, atol=FLOAT_TOL * lg.size)


def _check_trace(z, key, model, trace):
    checked = 0
    for layer in model.layers:
        rec = trace[layer.name]
        k_out, k_acc = f"{key}/{layer.name}/out_sha", f"{key}/{layer.name}/acc_sha"
        if k_out in z.files:
            assert sha(rec["out"].words) == _text(z, k_out), (key, layer.name, "out")
            checked += 1
        if k_acc in z.files:
            assert sha(rec["acc"]) == _text(z, k_acc), (key, layer.name, "acc")
            checked += 1
    want = sum(k.startswith(key + "/") and k.endswith(("/out_sha", "/acc_sha")) for k in z.files)
    assert checked == want and checked >= 50, (key, checked, want)  # every layer digest


def _traced(model, images, frames, dev):
    """One traced forward of the whole batch; per-frame traces sliced on the device."""
    n, h, w, _ = images.shape
    dm = DeviceModel(model, dev)
    ws_bytes = dm.plan(n, h, w, True)
    with torch.cuda.device(dev):
        ws = torch.empty(ws_bytes // 8 + 1, dtype=torch.int64, device=dev)
        img = torch.from_numpy(images).to(dev)
        logits = torch.empty((n, h, w, 1), dtype=torch.float64, device=dev)
        mask = torch.empty((n, h, w, 1), dtype=torch.uint8, device=dev)
        dm.run(img, logits, mask, ws)
        torch.cuda.synchronize(dev)
        out = {}
        for f in frames:
            lg = logits[f:f + 1].cpu().numpy()
            out[f] = (dm.read_trace(ws, lg, frames=slice(f, f + 1)), lg[0], mask[f].cpu().numpy())
        del ws, img, logits, mask
    torch.cuda.empty_cache()
    return out


def _engine(model, images, dev):
    eng = mb.Engine(model, batch=images.shape[0], device=dev)
    eng.image.copy_(torch.from_numpy(images))
    eng.run()
    torch.cuda.synchronize(dev)
    res = eng.logits.cpu().numpy(), eng.mask.cpu().numpy()
    del eng
    torch.cuda.empty_cache()
    return res


@pytest.fixture(scope="module")
def config3_images():
    return np.stack([bench_frame(i, 1024, 2048) for i in range(8)])


@pytest.mark.parametrize("gen", ["live0", "synth0"])
def test_config3_batch8_matches_reference(cuda, gen, config3_images):
    z = load_golden("forward_1024x2048.npz")
    model = _model(gen, 1024, 2048)
    got = _traced(model, config3_images, (0, 7), cuda)
    for f, (trace, lg, mk) in got.items():
        key = f"{gen}/f{f}"
        _check_outputs(z, key, lg, mk)
        _check_trace(z, key, model, trace)
    # the benchmarked executor (CUDA graph, fast epilogues, no trace)
    lg, mk = _engine(model, config3_images, cuda)
    for f in (0, 7):
        _check_outputs(z, f"{gen}/f{f}", lg[f], mk[f])


def test_config3_i8_engine_matches_reference(cuda, config3_images):
    """The kind::i8 cross-check engine (MBU_OPT_CONV_I8) at the bench shape."""
    z = load_golden("forward_1024x2048.npz")
    model = _model("live0", 1024, 2048)
    _lib.call("mbu_set_option", 3, 1)
    try:
        lg, mk = _engine(model, config3_images, cuda)
    finally:
        _lib.call("mbu_set_option", 3, 0)
    for f in (0, 7):
        _check_outputs(z, f"live0/f{f}", lg[f], mk[f])


def test_config5_4k_matches_reference(cuda):
    z = load_golden("forward_2160x3840.npz")
    model = _model("live0", 2160, 3840)
    images = bench_frame(0, 2160, 3840)[None]
    got = _traced(model, images, (0,), cuda)
    trace, lg, mk = got[0]
    _check_outputs(z, "live0/f0", lg, mk)
    _check_trace(z, "live0/f0", model, trace)
    lg, mk = _engine(model, images, cuda)
    _check_outputs(z, "live0/f0", lg[0], mk[0])
