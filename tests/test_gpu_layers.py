"""GPU parity of the layer operators (bit-exact) — runs on the B200 box.

Each case goes through the public layer API (``conv_forward`` etc., which
calls libmbunet through the C-ABI) and is compared with golden vectors the
reference produced, with the dense CPU oracle on fresh seeded inputs, and
across the two GPU execution paths (tcgen05 UTCIMMA and CUDA-core popcount).
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2601_11660_b200 as mb
from conftest import golden_cases
from oracle import dense
from paper_2601_11660_b200 import _lib

pytestmark = pytest.mark.gpu

PATHS = [_lib.PATH_AUTO, _lib.PATH_POPCOUNT]


@pytest.mark.parametrize("path", PATHS)
def test_conv_golden(cuda, path, conv_engine):
    z, cases = golden_cases()
    for c in cases:
        k = c["key"]
        if c["op"] == "conv":
            x = mb.pack_tensor(z[f"{k}_x"])
            planes = mb.pack_conv_weights(z[f"{k}_w"], x.segments, masked=c["masked"])
            spec = mb.ConvSpec(c["k"], c["k"], c["s"], c["p"], c["c_in"], c["c_out"],
                               pad_mode=c["pad_mode"])
            got = mb.conv_forward(x, planes, spec, path=path)
            assert got.dtype == np.int32
            assert np.array_equal(got, z[f"{k}_acc"]), k
        elif c["op"] == "gapconv":
            segs = tuple(mb.ChannelSegment(o, n) for o, n in c["segments"])
            words = z[f"{k}_words"]
            x = mb.BitTensor(1, words.shape[1], words.shape[2], 136, words, segs)
            planes = mb.pack_conv_weights(z[f"{k}_w"], segs, masked=c["masked"])
            got = mb.conv_forward(x, planes, mb.ConvSpec(3, 3, 1, 1, 136, 9), path=path)
            assert np.array_equal(got, z[f"{k}_acc"]), k


@pytest.mark.parametrize("path", PATHS)
def test_tconv_golden(cuda, path):
    z, cases = golden_cases()
    for c in cases:
        if c["op"] != "tconv":
            continue
        k = c["key"]
        x = mb.pack_tensor(z[f"{k}_x"])
        planes = mb.pack_conv_weights(z[f"{k}_w"], x.segments, masked=c["masked"])
        spec = mb.ConvSpec(c["k"], c["k"], c["k"], 0, c["c_in"], c["c_out"])
        got = mb.transposed_conv_forward(x, planes, spec, path=path)
        assert np.array_equal(got, z[f"{k}_acc"]), k


def test_pool_and_threshold_golden(cuda):
    z, cases = golden_cases()
    for c in cases:
        k = c["key"]
        if c["op"] == "pool":
            got = mb.maxpool2(mb.pack_tensor(z[f"{k}_x"]))
            assert np.array_equal(got.words, z[f"{k}_out"]), k
        elif c["op"] == "threshold":
            t = mb.FusedThreshold(z[f"{k}_t"], z[f"{k}_codes"])
            got = mb.apply_threshold(z[f"{k}_acc"], t)
            assert np.array_equal(got.words, z[f"{k}_out"]), k


def test_criterion3_random_layers_vs_oracle(cuda, rng, conv_engine):
    """Reference acceptance criterion 3 (test_acceptance.py:183-242), reduced."""
    pool = [64, 128, 192, 256]
    geoms = [(1, 1, 0), (2, 2, 0), (3, 1, 1), (3, 2, 1)]
    for trial in range(48):
        c_in = pool[trial % 4]
        c_out = int(rng.integers(1, 17)) if trial % 3 else pool[(trial // 4) % 4]
        k, s, p = geoms[trial % 4]
        masked = bool(trial % 2)
        h = w = 4 if s == 1 else 6
        x = rng.choice((-1, 1), size=(1, h, w, c_in)).astype(np.int8)
        wt = rng.choice((-1, 0, 1) if masked else (-1, 1), size=(c_out, k, k, c_in)).astype(np.int8)
        pad_mode = "zero" if masked and trial % 5 == 0 else "neg_one"
        xt = mb.pack_tensor(x)
        planes = mb.pack_conv_weights(wt, xt.segments, masked=masked)
        got = mb.conv_forward(xt, planes, mb.ConvSpec(k, k, s, p, c_in, c_out, pad_mode=pad_mode))
        ref = dense.ref_conv(x, wt, s, p, 0 if pad_mode == "zero" else -1)
        assert np.array_equal(got, ref), trial


@pytest.mark.parametrize("sparsity", [0.5, 0.9, 0.95])
def test_config2_conv_256_128x128(cuda, sparsity, conv_engine):
    """BASELINE config 2: one masked 3x3 conv 256->256 at 128x128, exact."""
    rng = np.random.default_rng(0)
    x = (rng.integers(0, 2, (1, 128, 128, 256)) * 2 - 1).astype(np.int8)
    nz = rng.random((256, 3, 3, 256)) >= sparsity
    wt = (nz * (rng.integers(0, 2, nz.shape) * 2 - 1)).astype(np.int8)
    xt = mb.pack_tensor(x)
    planes = mb.pack_conv_weights(wt, xt.segments, masked=True)
    spec = mb.ConvSpec(3, 3, 1, 1, 256, 256)
    got = mb.conv_forward(xt, planes, spec)
    assert _lib.last_path() == _lib.PATH_TCGEN05
    ref = dense.ref_conv(x, wt, 1, 1, -1)
    assert np.array_equal(got, ref)


def test_odd_channels_and_widths(cuda, rng, conv_engine):
    # partial 32-lane chunks, c_out not a multiple of 32, widths not multiples of 128
    for c_in, c_out, h, w in [(70, 9, 5, 7), (33, 40, 3, 130), (112, 64, 9, 33), (1, 1, 2, 2)]:
        x = rng.choice((-1, 1), size=(2, h, w, c_in)).astype(np.int8)
        wt = rng.choice((-1, 0, 1), size=(c_out, 3, 3, c_in)).astype(np.int8)
        xt = mb.pack_tensor(x)
        planes = mb.pack_conv_weights(wt, xt.segments, masked=True)
        for pad_mode in ("neg_one", "zero"):
            spec = mb.ConvSpec(3, 3, 1, 1, c_in, c_out, pad_mode=pad_mode)
            got = mb.conv_forward(xt, planes, spec)
            ref = dense.ref_conv(x, wt, 1, 1, 0 if pad_mode == "zero" else -1)
            assert np.array_equal(got, ref), (c_in, c_out, h, w, pad_mode)


def test_error_behaviour(cuda, rng):
    x = mb.pack_tensor(rng.choice((-1, 1), size=(1, 4, 4, 4)).astype(np.int8))
    wb = mb.pack_conv_weights(rng.choice((-1, 1), size=(2, 3, 3, 4)), x.segments, masked=False)
    with pytest.raises(mb.UnsupportedConfigError):
        mb.conv_forward(x, wb, mb.ConvSpec(3, 3, 1, 1, 4, 2, pad_mode="zero"))
    with pytest.raises(mb.ShapeError):
        mb.conv_forward(x, wb, mb.ConvSpec(3, 3, 1, 1, 5, 2))
    with pytest.raises(mb.LayoutError):
        mb.conv_forward(x, wb, mb.ConvSpec(3, 3, 1, 1, 4, 3))
    with pytest.raises(mb.UnsupportedConfigError):
        mb.transposed_conv_forward(x, wb, mb.ConvSpec(3, 3, 2, 0, 4, 2))


def test_float_endpoints_vs_oracle(cuda, rng):
    x = rng.random((2, 9, 11, 3))
    w = rng.normal(size=(64, 3, 3, 3))
    b = rng.normal(size=64)
    spec = mb.ConvSpec(3, 3, 1, 1, 3, 64)
    got = mb.float_conv(x, w, b, spec)
    assert np.allclose(got, dense.ref_float_conv(x, w, b, 1, 1), rtol=1e-12, atol=1e-12)
    g, be, m, v = rng.normal(size=64), rng.normal(size=64), rng.normal(size=64), rng.random(64)
    bits = mb.float_bn_sign(got, g, be, m, v, 1e-5)
    assert np.array_equal(mb.unpack_tensor(bits), dense.ref_bn_sign(got, g, be, m, v, 1e-5))


def test_bit_gemm_vs_numpy(cuda, rng):
    a = mb.PackedBitMatrix.pack_rows(rng.choice((-1, 1), size=(37, 256)))
    pos, neg = mb.PackedBitMatrix.pack_ternary_rows(rng.choice((-1, 0, 1), size=(11, 256)))
    dense_a = 2 * np.unpackbits(a.words.view(np.uint8), bitorder="little").reshape(37, 256).astype(np.int64) - 1
    pb = np.unpackbits(pos.words.view(np.uint8), bitorder="little").reshape(11, 256).astype(np.int64)
    nb = np.unpackbits(neg.words.view(np.uint8), bitorder="little").reshape(11, 256).astype(np.int64)
    assert np.array_equal(mb.bit_gemm(a, pos, neg, 256), dense_a @ (pb - nb).T)


def _stem_bits(fc, x, cuda, mode):
    """Run a stem FloatConvHandle in one of its three execution modes:
    "tc" (tcgen05 bf16-split + float64 recheck), "ffma" (float32 CUDA cores +
    float64 recheck) or "generic" (all float64)."""
    import torch

    n, h, w, _ = x.shape
    generic, ffma = {"tc": (0, 0), "ffma": (0, 1), "generic": (1, 0)}[mode]
    _lib.call("mbu_set_option", 1, generic)
    _lib.call("mbu_set_option", 2, ffma)
    try:
        out = torch.zeros((n, h, w, 2), dtype=torch.int64, device=cuda)
        fc.run(n, h, w, x_f64=torch.from_numpy(x).to(cuda), bits=out)
        torch.cuda.synchronize()
    finally:
        _lib.call("mbu_set_option", 1, 0)
        _lib.call("mbu_set_option", 2, 0)
    return out.cpu().numpy()


def test_stem_fast_path_equals_float64_path(cuda):
    """The tensor-core and float32 stems (both with exact float64 re-check)
    must reproduce the all-float64 kernel bit for bit, including pixels
    planted exactly on the batchnorm decision boundary (which force the
    re-check), a non-finite input and a constant (gamma = 0) channel."""
    from paper_2601_11660_b200.ops import FloatConvHandle

    rng = np.random.default_rng(5)
    x = rng.random((2, 40, 136, 3))
    x[0, 3, 4] = [np.inf, 0.5, 0.5]  # non-finite input goes down the exact path
    w = rng.normal(size=(64, 3, 3, 3))
    b = rng.normal(size=64)
    g = rng.uniform(-1.5, 1.5, 64)
    g[0] = 0.0
    be = rng.normal(size=64)
    v = rng.uniform(0.5, 2.0, 64)
    eps = 1e-5
    acc = dense.ref_float_conv(x[1:2], w, b, 1, 1)
    sigma = np.sqrt(v + eps)
    mean = acc[0, 17, 9, :] + be * sigma / np.where(g == 0, 1.0, g)  # boundary on a pixel
    spec = mb.ConvSpec(3, 3, 1, 1, 3, 64)
    fc = FloatConvHandle(w, b, spec, bn=(g, be, mean, v, eps))
    outs = [_stem_bits(fc, x, cuda, m) for m in ("tc", "ffma", "generic")]
    assert np.array_equal(outs[0], outs[2])
    assert np.array_equal(outs[1], outs[2])
    ref = dense.ref_bn_sign(dense.ref_float_conv(x, w, b, 1, 1), g, be, mean, v, eps)
    got = mb.unpack_tensor(mb.BitTensor(2, 40, 136, 64, outs[0].view(np.uint64)))
    diff = got != ref
    assert diff.sum() <= 64, diff.sum()  # only planted exact-boundary pixels may round differently


@pytest.mark.parametrize("shape", [(1, 37, 258), (2, 64, 128), (1, 5, 6)])
def test_stem_tc_exact_ties(cuda, shape):
    """Dyadic inputs and weights make the stem accumulator exact, and the
    batchnorm means are set to accumulator values that occur, so a large
    share of decisions lands exactly on (or one rounding away from) the
    boundary: every one of them must be re-decided in float64 and agree with
    the all-float64 kernel. Odd tile remainders (H % 4, W % 128) included."""
    from paper_2601_11660_b200.ops import FloatConvHandle

    rng = np.random.default_rng(77)
    x = rng.integers(0, 8, size=shape + (3,)) / 8.0
    w = rng.integers(-2, 3, size=(64, 3, 3, 3)) / 4.0
    b = rng.integers(-4, 5, size=64) / 16.0
    g = np.where(rng.random(64) < 0.5, 1.0, -1.0)
    be = np.zeros(64)
    v = np.ones(64)
    acc = dense.ref_float_conv(x, w, b, 1, 1).reshape(-1, 64)
    mean = acc[rng.integers(0, acc.shape[0], 64), np.arange(64)]
    mean[::7] += 2.0 ** -40  # one rounding away from a reachable value
    fc = FloatConvHandle(w, b, mb.ConvSpec(3, 3, 1, 1, 3, 64), bn=(g, be, mean, v, 0.0))
    tc = _stem_bits(fc, x, cuda, "tc")
    gen = _stem_bits(fc, x, cuda, "generic")
    assert np.array_equal(tc, gen)
    ref = dense.ref_bn_sign(dense.ref_float_conv(x, w, b, 1, 1), g, be, mean, v, 0.0)
    got = mb.unpack_tensor(mb.BitTensor(*shape, 64, tc.view(np.uint64)))
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("c_in,c_out", [(512, 384), (256, 512), (128, 96)])
def test_wide_tconv_row_mode_vs_oracle(cuda, rng, c_in, c_out):
    """2x2/s2 tconvs whose output taps exceed one 256-column N tile (up-CT1:
    384 channels, tiles that straddle two taps) at row-mode widths (>= 128
    columns, including a ragged column tile) against the dense oracle."""
    for h, w in [(2, 128), (3, 136)]:
        x = rng.choice((-1, 1), size=(2, h, w, c_in)).astype(np.int8)
        wt = rng.choice((-1, 0, 1), size=(c_out, 2, 2, c_in)).astype(np.int8)
        xt = mb.pack_tensor(x)
        planes = mb.pack_conv_weights(wt, xt.segments, masked=True)
        spec = mb.ConvSpec(2, 2, 2, 0, c_in, c_out)
        got = mb.transposed_conv_forward(xt, planes, spec)
        ref = dense.ref_tconv(x, wt, 2)
        assert np.array_equal(got, ref), (c_in, c_out, h, w)
