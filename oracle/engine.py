"""Packed CPU engine port — TEST INFRASTRUCTURE / CPU BASELINE ONLY.

A restatement of the reference's own CPU execution path for the forward
call: ``graph.forward`` (``pkg/src/bitunet/graph.py:413-458``) interpreting
the layer list, ``conv_forward`` (``layers.py:289-313``) lowering to im2row
over packed words (``layers.py:258-277``), ``bit_gemm`` (``bitcore.py:265-294``)
in its XOR forms, ``xor_popcount_rows`` (``kernels.py:114-147``, here the C
loop of ``oracle/xorpop.c``), ``apply_threshold`` (``layers.py:508-522``),
``maxpool2``/``concat_channels`` (``layers.py:360-384``) and the float64
stem/head (``layers.py:530-560``, per-tap BLAS like the reference).

It works on plain arrays: a bit tensor is ``(words, segments)`` with words
shaped (n, h, w, wpp) uint64 and segments a tuple of (lane_offset, count).
It consumes any model object with the reference's attribute names.
``bench.py`` times it as the CPU baseline (``kind = "port"``); the tests use
it as a second, layout-level oracle (its words must equal the GPU's
byte-for-byte).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import build as _build

DIR_GE, DIR_LE, CONST_NEG, CONST_POS = 0, 1, 2, 3


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def xor_popcount_rows(a, b, threads=1):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    out = np.empty((a.shape[0], b.shape[0]), dtype=np.int32)
    if out.size:
        _build.load().oracle_xor_popcount_rows(
            a.ctypes.data_as(ctypes.c_void_p), b.ctypes.data_as(ctypes.c_void_p),
            out.ctypes.data_as(ctypes.c_void_p), a.shape[0], b.shape[0], a.shape[1], threads)
    return out


def _lanes(segments):
    end = max((o + c for o, c in segments), default=0)
    return -(-end // 128) * 128


def _segs(obj):
    return tuple((int(s.lane_offset), int(s.count)) for s in obj)


def _plane_rows(weights, rows, width):
    masked = hasattr(weights, "neg")
    first = weights.pos if masked else weights
    pos = np.asarray(first.words).reshape(rows, width)
    neg = np.asarray(weights.neg.words).reshape(rows, width) if masked else None
    return pos, neg


def bit_gemm(a, pos, neg, k_true, threads):
    if neg is not None:
        return xor_popcount_rows(a, neg, threads) - xor_popcount_rows(a, pos, threads)
    return (np.int32(k_true) - 2 * xor_popcount_rows(a, pos, threads)).astype(np.int32)


def conv_forward(words, segments, weights, spec, threads=1):
    n, h, w, wpp = words.shape
    c = sum(cnt for _, cnt in segments)
    kh, kw, s, p = spec.kernel_h, spec.kernel_w, spec.stride, spec.padding
    ho = (h + 2 * p - kh) // s + 1
    wo = (w + 2 * p - kw) // s + 1
    xp = np.pad(words, ((0, 0), (p, p), (p, p), (0, 0))) if p else words
    cols = np.empty((n, ho, wo, kh, kw, wpp), dtype=np.uint64)
    for dy in range(kh):
        for dx in range(kw):
            cols[:, :, :, dy, dx, :] = xp[:, dy:dy + s * ho:s, dx:dx + s * wo:s, :]
    a = cols.reshape(n * ho * wo, kh * kw * wpp)
    pos, neg = _plane_rows(weights, spec.c_out, kh * kw * wpp)
    acc = bit_gemm(a, pos, neg, kh * kw * c, threads).reshape(n, ho, wo, spec.c_out)
    if spec.pad_mode == "zero" and p > 0:
        pc = np.bitwise_count(pos.reshape(spec.c_out, kh * kw, wpp)).sum(axis=2, dtype=np.int64)
        if neg is not None:
            pc = pc - np.bitwise_count(neg.reshape(spec.c_out, kh * kw, wpp)).sum(axis=2, dtype=np.int64)
        ry = np.arange(ho)[:, None] * s - p + np.arange(kh)[None, :]
        rx = np.arange(wo)[:, None] * s - p + np.arange(kw)[None, :]
        oob = ((ry < 0) | (ry >= h))[:, None, :, None] | ((rx < 0) | (rx >= w))[None, :, None, :]
        corr = np.tensordot(oob.astype(np.int64), pc.reshape(spec.c_out, kh, kw), axes=([2, 3], [1, 2]))
        acc = (acc + corr[None]).astype(np.int32)
    return acc


def transposed_conv_forward(words, segments, weights, spec, threads=1):
    n, h, w, wpp = words.shape
    c = sum(cnt for _, cnt in segments)
    s = spec.stride
    pos, neg = _plane_rows(weights, spec.c_out, s * s * wpp)
    pos = pos.reshape(spec.c_out, s * s, wpp)
    neg = None if neg is None else neg.reshape(spec.c_out, s * s, wpp)
    a = words.reshape(n * h * w, wpp)
    out = np.empty((n, h * s, w * s, spec.c_out), dtype=np.int32)
    for dy in range(s):
        for dx in range(s):
            t = dy * s + dx
            acc = bit_gemm(a, np.ascontiguousarray(pos[:, t]),
                           None if neg is None else np.ascontiguousarray(neg[:, t]), c, threads)
            out[:, dy::s, dx::s, :] = acc.reshape(n, h, w, spec.c_out)
    return out


def pack_bool(bits):
    n, h, w, c = bits.shape
    lanes = -(-c // 128) * 128
    full = np.zeros((n, h, w, lanes), dtype=np.uint8)
    full[..., :c] = bits
    words = np.packbits(full, axis=-1, bitorder="little").view("<u8").astype(np.uint64)
    return words, ((0, c),)


def apply_threshold(acc, threshold):
    t = np.asarray(threshold.thresholds, dtype=np.int32)
    codes = np.asarray(threshold.codes)
    bits = np.where(codes == DIR_GE, acc >= t, np.where(codes == DIR_LE, acc <= t, codes == CONST_POS))
    return pack_bool(bits)


def maxpool2(words):
    n, h, w, wpp = words.shape
    v = words.reshape(n, h // 2, 2, w // 2, 2, wpp)
    return v[:, :, 0, :, 0] | v[:, :, 0, :, 1] | v[:, :, 1, :, 0] | v[:, :, 1, :, 1]


def concat(a, b):
    (wa, sa), (wb, sb) = a, b
    shift = _lanes(sa)
    return np.concatenate([wa, wb], axis=-1), sa + tuple((o + shift, c) for o, c in sb)


def unpack(words, segments):
    bits = np.unpackbits(np.ascontiguousarray(words, dtype="<u8").view(np.uint8), axis=-1,
                         bitorder="little")
    lanes = np.concatenate([o + np.arange(c) for o, c in segments])
    return 2 * bits[..., lanes].astype(np.int8) - 1


def float_conv(x, w, bias, spec):
    x = np.asarray(x, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    n, h, wd, ci = x.shape
    s, p = spec.stride, spec.padding
    ho = (h + 2 * p - spec.kernel_h) // s + 1
    wo = (wd + 2 * p - spec.kernel_w) // s + 1
    xp = np.zeros((n, h + 2 * p, wd + 2 * p, ci))
    xp[:, p:p + h, p:p + wd, :] = x
    out = np.zeros((n, ho, wo, spec.c_out))
    for dy in range(spec.kernel_h):
        for dx in range(spec.kernel_w):
            out += xp[:, dy:dy + s * ho:s, dx:dx + s * wo:s, :] @ w[:, dy, dx, :].T
    if bias is not None:
        out += np.asarray(bias, dtype=np.float64)
    return out


def bn_sign(acc, gamma, beta, mean, var, eps, bias=None):
    sigma = np.sqrt(np.asarray(var, np.float64) + eps)
    pre = acc + (0.0 if bias is None else np.asarray(bias, np.float64))
    y = np.asarray(gamma, np.float64) * (pre - np.asarray(mean, np.float64)) / sigma
    return pack_bool(y + np.asarray(beta, np.float64) >= 0.0)


def forward(model, image, threads=1, trace=False):
    """Run a compiled model; returns (logits, mask, trace-or-None).

    Trace entries are {"acc": ..., "out": words | float array} like the
    reference's, with bit outputs as raw (n, h, w, wpp) uint64 words.
    """
    image = np.asarray(image, dtype=np.float64)
    outs = {}
    notes = {} if trace else None
    x = image  # float array or (words, segments)
    logits = None
    for layer in model.layers:
        acc = None
        kind = layer.kind
        if kind == "float-conv":
            dense = unpack(*x).astype(np.float64) if isinstance(x, tuple) else x
            acc = float_conv(dense, layer.weights, layer.bias, layer.spec)
            if layer.apply_sign:
                x = bn_sign(acc, *layer.bn)
            else:
                x = logits = acc
        elif kind in ("binary-conv", "masked-conv"):
            acc = conv_forward(x[0], x[1], layer.weights, layer.spec, threads)
            x = apply_threshold(acc, layer.threshold)
        elif kind in ("binary-tconv", "masked-tconv"):
            acc = transposed_conv_forward(x[0], x[1], layer.weights, layer.spec, threads)
            x = apply_threshold(acc, layer.threshold)
        elif kind == "maxpool":
            x = (maxpool2(x[0]), x[1])
        elif kind == "concat":
            x = concat(x, outs[layer.concat_with])
        outs[layer.name] = x
        if notes is not None:
            notes[layer.name] = {"acc": acc, "out": x[0] if isinstance(x, tuple) else x}
    mask = (logits >= 0.0).astype(np.uint8)
    if notes is not None:
        notes["mask"] = mask
    return logits, mask, notes
