"""Layer descriptions and build-time producers of the weight layout.

Host-side restatement of the non-arithmetic half of
``pkg/src/bitunet/layers.py``: :class:`ConvSpec` (``:76-101``),
:class:`FusedThreshold` and its codes (``:66-70``, ``:104-127``), plane
packing (``pack_conv_weights`` ``:147-182`` / ``unpack_conv_weights``
``:185-213``), per-position weight sums (``:236-250``) and BN folding
(``fuse_bn_sign`` ``:455-505``). These run once per model build.

The data-parallel operators of the reference module (``conv_forward``,
``transposed_conv_forward``, ``apply_threshold``, ``maxpool2``,
``float_conv``, ``float_bn_sign``) are re-exported from
:mod:`paper_2601_11660_b200.ops`, where they execute on sm_100a through
``libmbunet.so``; ``concat_channels`` is a pure lane-layout operation.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .bitcore import (
    WORD_BITS,
    BitPlane,
    BitTensor,
    ChannelSegment,
    MaskedWeightPlanes,
    bits_to_words,
    is_masked,
    segment_lane_table,
    segment_lanes,
    words_to_bits,
)
from .errors import LayoutError, ShapeError, UnsupportedConfigError, ValueAlphabetError

__all__ = [
    "DIR_GE",
    "DIR_LE",
    "CONST_NEG",
    "CONST_POS",
    "ConvSpec",
    "FusedThreshold",
    "segment_lanes",
    "segment_lane_table",
    "pack_conv_weights",
    "unpack_conv_weights",
    "weight_position_sums",
    "fuse_bn_sign",
    "concat_channels",
]

# threshold codes; also the serialized values (layers.py:66-70)
DIR_GE = 0
DIR_LE = 1
CONST_NEG = 2
CONST_POS = 3

INT32_MIN = -(2**31)
INT32_MAX = 2**31 - 1


@dataclass(frozen=True)
class ConvSpec:
    """Convolution geometry (``layers.py:76-101``)."""

    kernel_h: int
    kernel_w: int
    stride: int
    padding: int
    c_in: int
    c_out: int
    pad_mode: str = "neg_one"

    def __post_init__(self):
        if min(self.kernel_h, self.kernel_w, self.stride) < 1:
            raise ShapeError(f"kernel and stride must be >= 1: {self}")
        if self.padding < 0 or min(self.c_in, self.c_out) < 1:
            raise ShapeError(f"padding or channel count out of range: {self}")
        if self.pad_mode not in ("neg_one", "zero"):
            raise UnsupportedConfigError(f"unknown pad_mode {self.pad_mode!r}")

    def out_extent(self, h: int, w: int) -> tuple:
        ho = (h + 2 * self.padding - self.kernel_h) // self.stride + 1
        wo = (w + 2 * self.padding - self.kernel_w) // self.stride + 1
        if ho <= 0 or wo <= 0:
            raise ShapeError(f"kernel larger than the padded input: {self} on {h}x{w}")
        return ho, wo


@dataclass(frozen=True, eq=False)
class FusedThreshold:
    """Per-channel integer stand-in for BN + bias + sign (``layers.py:104-127``)."""

    thresholds: np.ndarray
    codes: np.ndarray

    def __post_init__(self):
        t = np.ascontiguousarray(self.thresholds, dtype=np.int32)
        c = np.ascontiguousarray(self.codes, dtype=np.uint8)
        object.__setattr__(self, "thresholds", t)
        object.__setattr__(self, "codes", c)
        if t.ndim != 1 or t.shape != c.shape:
            raise ShapeError(f"thresholds {t.shape} and codes {c.shape} must be matching vectors")
        if c.size and int(c.max()) > CONST_POS:
            raise ValueAlphabetError(f"unknown threshold code {int(c.max())}")

    @property
    def n_channels(self) -> int:
        return self.thresholds.shape[0]


# --------------------------------------------------------------------------- #
# weight planes
# --------------------------------------------------------------------------- #


def _tap_lane_index(kh: int, kw: int, segments) -> np.ndarray:
    """Flat K-lane of (tap, channel) for the documented weight order."""
    lpp = segment_lanes(segments)
    taps = np.arange(kh * kw, dtype=np.int64)[:, None] * lpp
    return (taps + segment_lane_table(segments)[None, :]).reshape(-1)


def pack_conv_weights(w, segments, masked: bool):
    """Dense (c_out, kh, kw, c_in) -> flat planes in the input's lane layout.

    Lane of weight (o, dy, dx, j) = o*K + (dy*kw + dx)*lpp + lane_j, with
    K = kh*kw*lpp and lane_j the input lane of channel j (``layers.py:147-182``).
    """
    w = np.asarray(w)
    if w.ndim != 4:
        raise ShapeError(f"expected (c_out, k_h, k_w, c_in) weights, got {w.shape}")
    co, kh, kw, ci = w.shape
    if ci != sum(s.count for s in segments):
        raise ShapeError(f"weight c_in {ci} != {sum(s.count for s in segments)} segment channels")
    allowed = (-1, 0, 1) if masked else (-1, 1)
    if w.size and not np.isin(w, allowed).all():
        raise ValueAlphabetError(f"weights outside {allowed}")
    k_lanes = kh * kw * segment_lanes(segments)
    lanes = _tap_lane_index(kh, kw, segments)
    flat = w.reshape(co, -1)

    def plane(sel) -> BitPlane:
        bits = np.zeros((co, k_lanes), dtype=np.uint8)
        bits[:, lanes] = sel
        return BitPlane(co * k_lanes, bits_to_words(bits).reshape(-1))

    if masked:
        return MaskedWeightPlanes(plane(flat > 0), plane(flat < 0))
    return plane(flat > 0)


def unpack_conv_weights(weights, spec: ConvSpec, segments) -> np.ndarray:
    """Planes -> dense int8 (c_out, kh, kw, c_in) (``layers.py:185-213``)."""
    co, kh, kw = spec.c_out, spec.kernel_h, spec.kernel_w
    k_lanes = kh * kw * segment_lanes(segments)
    masked = is_masked(weights)
    first = weights.pos if masked else weights
    if first.n_bits != co * k_lanes:
        raise LayoutError(f"weight plane has {first.n_bits} lanes, expected {co}*{k_lanes}")
    lanes = _tap_lane_index(kh, kw, segments)
    ci = sum(s.count for s in segments)

    def bits(p) -> np.ndarray:
        return words_to_bits(np.asarray(p.words).reshape(co, k_lanes // WORD_BITS)).astype(np.int8)

    vals = bits(first) - bits(weights.neg) if masked else 2 * bits(first) - 1
    return vals[:, lanes].reshape(co, kh, kw, ci)


def weight_position_sums(weights, c_out: int, kh: int, kw: int, lanes_per_pixel: int) -> np.ndarray:
    """Signed sum of each (out channel, tap) weight slice (``layers.py:236-250``)."""
    masked = is_masked(weights)
    first = weights.pos if masked else weights
    shape = (c_out, kh * kw, lanes_per_pixel // WORD_BITS)
    s = np.bitwise_count(np.asarray(first.words).reshape(shape)).sum(axis=2, dtype=np.int64)
    if masked:
        s = s - np.bitwise_count(np.asarray(weights.neg.words).reshape(shape)).sum(
            axis=2, dtype=np.int64
        )
    return s.reshape(c_out, kh, kw).astype(np.int32)


# --------------------------------------------------------------------------- #
# batchnorm folding (build time)
# --------------------------------------------------------------------------- #


def _bn_fires(a, gamma, beta, mean, sigma, bias):
    """The float64 decision the fused threshold reproduces (``layers.py:392-395``).

    Evaluated in exactly the reference's operation order.
    """
    pre = a + bias
    return gamma * (pre - mean) / sigma + beta >= 0.0


def fuse_bn_sign(gamma, beta, mean, var, eps, bias=None) -> FusedThreshold:
    """Fold BN + bias + sign into exact int32 thresholds (``layers.py:455-505``).

    For gamma > 0 the output bit is ``acc >= T`` with T the smallest int32
    for which the float predicate fires; for gamma < 0 it is ``acc <= T``
    with T the largest such int32; gamma == 0 is a constant. The float
    predicate is monotone in ``acc`` (every step is a rounded monotone map),
    so T is unique and a vectorised bisection over the int32 range finds the
    same T as the reference's snap-then-refine search.
    """
    gamma = np.asarray(gamma, dtype=np.float64)
    beta = np.asarray(beta, dtype=np.float64)
    mean = np.asarray(mean, dtype=np.float64)
    var = np.asarray(var, dtype=np.float64)
    c = gamma.shape[0]
    if not (beta.shape == mean.shape == var.shape == (c,)):
        raise ShapeError("batchnorm vectors must share one channel axis")
    bias = np.zeros(c) if bias is None else np.asarray(bias, dtype=np.float64)
    if bias.shape != (c,):
        raise ShapeError(f"bias shape {bias.shape} != ({c},)")
    if np.any(var < 0):
        raise ValueAlphabetError("variance must be nonnegative")
    if not np.isfinite(np.stack([gamma, beta, mean, var, bias])).all() or not (
        eps > 0 and np.isfinite(eps)
    ):
        raise ValueAlphabetError("batchnorm parameters must be finite with eps > 0")
    sigma = np.sqrt(var + eps)

    def fires(a, sel):
        return _bn_fires(
            a.astype(np.float64), gamma[sel], beta[sel], mean[sel], sigma[sel], bias[sel]
        )

    thresholds = np.zeros(c, dtype=np.int64)
    codes = np.full(c, CONST_NEG, dtype=np.uint8)
    codes[(gamma == 0.0) & (beta >= 0.0)] = CONST_POS

    up = np.flatnonzero(gamma > 0.0)
    if up.size:
        live = fires(np.full(up.size, INT32_MAX, dtype=np.int64), up)
        up = up[live]
    if up.size:  # smallest true T: pred(hi) true, pred(lo) false (lo may be virtual)
        lo = np.full(up.size, INT32_MIN - 1, dtype=np.int64)
        hi = np.full(up.size, INT32_MAX, dtype=np.int64)
        for _ in range(34):
            mid = (lo + hi) // 2
            ok = fires(mid, up) & (hi - lo > 1)
            hi = np.where(ok, mid, hi)
            lo = np.where(ok | (hi - lo <= 1), lo, mid)
        thresholds[up] = hi
        codes[up] = DIR_GE

    down = np.flatnonzero(gamma < 0.0)
    if down.size:
        live = fires(np.full(down.size, INT32_MIN, dtype=np.int64), down)
        down = down[live]
    if down.size:  # largest true T: pred(lo) true, pred(hi) false (hi may be virtual)
        lo = np.full(down.size, INT32_MIN, dtype=np.int64)
        hi = np.full(down.size, INT32_MAX + 1, dtype=np.int64)
        for _ in range(34):
            mid = (lo + hi) // 2
            ok = fires(mid, down) & (hi - lo > 1)
            lo = np.where(ok, mid, lo)
            hi = np.where(ok | (hi - lo <= 1), hi, mid)
        thresholds[down] = lo
        codes[down] = DIR_LE
    return FusedThreshold(thresholds.astype(np.int32), codes)


# --------------------------------------------------------------------------- #
# concat (lane layout only)
# --------------------------------------------------------------------------- #


def concat_channels(a, b):
    """Word concatenation, ``b`` at a fresh 128-lane block (``layers.py:369-384``).

    A pure layout operation with no arithmetic. Inside the GPU forward it
    costs nothing: the producers of both operands write straight into their
    word ranges of one shared buffer (see ``graph.forward``).
    """
    if (a.n, a.h, a.w) != (b.n, b.h, b.w):
        raise ShapeError(f"spatial extents differ: {(a.n, a.h, a.w)} vs {(b.n, b.h, b.w)}")
    if b.c == 0:
        return a
    if a.c == 0:
        return b
    shift = a.lanes_per_pixel
    segs = tuple(a.segments) + tuple(
        ChannelSegment(s.lane_offset + shift, s.count) for s in b.segments
    )
    words = np.concatenate([np.asarray(a.words), np.asarray(b.words)], axis=-1)
    return BitTensor(a.n, a.h, a.w, a.c + b.c, words, segs)
