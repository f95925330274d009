"""Packed bit containers: the layout contract of the drop-in boundary.

These are host-side restatements of the reference containers in
``pkg/src/bitunet/bitcore.py`` (layout doc ``:3-18``). They hold NumPy
arrays exactly as the reference does, so a ``BitTensor.words`` array produced
by the GPU path compares byte-for-byte with the reference's.

Encoding (unchanged from the reference):

* a bipolar value a in {-1,+1} is the bit a' = (a+1)/2 (1 means +1);
* lane i of a pixel lives at bit (i % 64) of uint64 word (i // 64),
  LSB first; channels are grouped into 128-lane blocks;
* a ternary weight b = pos - neg with pos AND neg == 0;
* pad lanes are 0 in activations and in both weight planes.

The arithmetic of the hot path (``bit_gemm`` and everything above it) runs
on the GPU; see :mod:`paper_2601_11660_b200.ops`. Functions here only pack,
unpack and validate.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import LayoutError, PlaneOverlapError, ShapeError, ValueAlphabetError

WORD_BITS = 64
BLOCK_BITS = 128
WORDS_PER_BLOCK = BLOCK_BITS // WORD_BITS

__all__ = [
    "WORD_BITS",
    "BLOCK_BITS",
    "WORDS_PER_BLOCK",
    "BitPlane",
    "MaskedWeightPlanes",
    "PackedBitMatrix",
    "ChannelSegment",
    "BitTensor",
    "pack_bipolar",
    "unpack_bipolar",
    "pack_tensor",
    "pack_bits_tensor",
    "unpack_tensor",
    "bits_to_words",
    "words_to_bits",
    "is_masked",
]


def _n_words(n_bits: int) -> int:
    return (n_bits + WORD_BITS - 1) // WORD_BITS


def _round_block(lanes: int) -> int:
    return ((lanes + BLOCK_BITS - 1) // BLOCK_BITS) * BLOCK_BITS


def bits_to_words(bits: np.ndarray) -> np.ndarray:
    """(..., L) 0/1 -> (..., L/64) uint64, lane i at bit i%64 (L % 64 == 0)."""
    b = np.ascontiguousarray(bits, dtype=np.uint8)
    if b.shape[-1] % WORD_BITS:
        raise LayoutError(f"{b.shape[-1]} lanes is not a whole number of words")
    packed = np.packbits(b, axis=-1, bitorder="little")
    return np.ascontiguousarray(packed).view("<u8").astype(np.uint64, copy=False)


def words_to_bits(words: np.ndarray) -> np.ndarray:
    """Inverse of :func:`bits_to_words`: (..., W) uint64 -> (..., 64W) uint8."""
    w = np.ascontiguousarray(words, dtype="<u8")
    return np.unpackbits(w.view(np.uint8), axis=-1, bitorder="little")


def _final_word_mask(n_bits: int) -> int:
    r = n_bits % WORD_BITS
    return (1 << WORD_BITS) - 1 if r == 0 else (1 << r) - 1


@dataclass(frozen=True, eq=False)
class BitPlane:
    """``n_bits`` bipolar lanes packed into uint64 words (``bitcore.py:83-102``)."""

    n_bits: int
    words: np.ndarray

    def __post_init__(self):
        w = np.ascontiguousarray(self.words, dtype=np.uint64)
        object.__setattr__(self, "words", w)
        if self.n_bits < 0:
            raise LayoutError(f"negative lane count {self.n_bits}")
        if w.ndim != 1 or w.shape[0] != _n_words(self.n_bits):
            raise LayoutError(
                f"{self.n_bits} lanes need {_n_words(self.n_bits)} words, got shape {w.shape}"
            )
        if w.size and self.n_bits % WORD_BITS:
            if int(w[-1]) & ~_final_word_mask(self.n_bits):
                raise LayoutError("lanes past n_bits must be zero")


@dataclass(frozen=True, eq=False)
class MaskedWeightPlanes:
    """Subtractive ternary planes, value = pos - neg (``bitcore.py:105-122``)."""

    pos: BitPlane
    neg: BitPlane

    def __post_init__(self):
        if self.pos.n_bits != self.neg.n_bits:
            raise LayoutError(
                f"plane lane counts differ: {self.pos.n_bits} vs {self.neg.n_bits}"
            )
        if np.any(self.pos.words & self.neg.words):
            raise PlaneOverlapError("a lane is set in both pos and neg")

    @property
    def n_bits(self) -> int:
        return self.pos.n_bits


def is_masked(weights) -> bool:
    """Duck-typed ``isinstance(weights, MaskedWeightPlanes)``.

    Accepts the reference's own classes as well as ours, which is what makes
    the GPU path a drop-in for models built by ``bitunet.build``.
    """
    return hasattr(weights, "pos") and hasattr(weights, "neg")


def pack_bipolar(values) -> BitPlane:
    v = np.asarray(values).reshape(-1)
    if v.size == 0:
        return BitPlane(0, np.zeros(0, dtype=np.uint64))
    if not np.isin(v, (-1, 1)).all():
        raise ValueAlphabetError("pack_bipolar expects values in {-1,+1}")
    lanes = _n_words(v.size) * WORD_BITS
    bits = np.zeros(lanes, dtype=np.uint8)
    bits[: v.size] = v > 0
    return BitPlane(v.size, bits_to_words(bits))


def unpack_bipolar(plane: BitPlane) -> np.ndarray:
    if plane.n_bits == 0:
        return np.zeros(0, dtype=np.int8)
    bits = words_to_bits(plane.words)[: plane.n_bits].astype(np.int8)
    return 2 * bits - 1


@dataclass(frozen=True, eq=False)
class PackedBitMatrix:
    """R packed rows of ``n_lanes`` lanes (``bitcore.py:211-262``)."""

    n_lanes: int
    words: np.ndarray

    def __post_init__(self):
        w = np.ascontiguousarray(self.words, dtype=np.uint64)
        object.__setattr__(self, "words", w)
        if w.ndim != 2 or w.shape[1] != _n_words(self.n_lanes):
            raise LayoutError(
                f"{self.n_lanes} lanes need rows of {_n_words(self.n_lanes)} words, "
                f"got shape {w.shape}"
            )
        if w.size and self.n_lanes % WORD_BITS:
            tail = np.uint64(~_final_word_mask(self.n_lanes) & ((1 << 64) - 1))
            if np.any(w[:, -1] & tail):
                raise LayoutError("lanes past n_lanes must be zero")

    @property
    def n_rows(self) -> int:
        return self.words.shape[0]

    @classmethod
    def pack_rows(cls, values: np.ndarray) -> "PackedBitMatrix":
        v = np.asarray(values)
        if v.ndim != 2:
            raise ShapeError(f"expected 2-d rows, got shape {v.shape}")
        if v.size and not np.isin(v, (-1, 1)).all():
            raise ValueAlphabetError("pack_rows expects values in {-1,+1}")
        r, n = v.shape
        bits = np.zeros((r, _n_words(n) * WORD_BITS), dtype=np.uint8)
        bits[:, :n] = v > 0
        return cls(n, bits_to_words(bits))

    @classmethod
    def pack_ternary_rows(cls, values: np.ndarray):
        v = np.asarray(values)
        if v.ndim != 2:
            raise ShapeError(f"expected 2-d rows, got shape {v.shape}")
        if v.size and not np.isin(v, (-1, 0, 1)).all():
            raise ValueAlphabetError("pack_ternary_rows expects values in {-1,0,+1}")
        r, n = v.shape
        lanes = _n_words(n) * WORD_BITS
        pos = np.zeros((r, lanes), dtype=np.uint8)
        neg = np.zeros((r, lanes), dtype=np.uint8)
        pos[:, :n] = v > 0
        neg[:, :n] = v < 0
        return cls(n, bits_to_words(pos)), cls(n, bits_to_words(neg))


@dataclass(frozen=True)
class ChannelSegment:
    """``count`` channels starting at pixel lane ``lane_offset`` (``bitcore.py:302-311``)."""

    lane_offset: int
    count: int


@dataclass(frozen=True, eq=False)
class BitTensor:
    """(n, h, w, c) bipolar tensor packed per pixel (``bitcore.py:314-388``).

    ``words`` has shape (n, h, w, words_per_pixel). Channels occupy the lanes
    named by ``segments``; every other lane is zero.
    """

    n: int
    h: int
    w: int
    c: int
    words: np.ndarray
    segments: tuple = field(default=())

    def __post_init__(self):
        words = np.ascontiguousarray(self.words, dtype=np.uint64)
        object.__setattr__(self, "words", words)
        segs = tuple(self.segments)
        if not segs and self.c:
            segs = (ChannelSegment(0, self.c),)
        object.__setattr__(self, "segments", segs)
        if sum(s.count for s in segs) != self.c:
            raise LayoutError(f"segments hold {sum(s.count for s in segs)} channels, c={self.c}")
        prev_end = 0
        for s in segs:
            if s.count <= 0 or s.lane_offset % BLOCK_BITS:
                raise LayoutError(f"segment {s} must be block aligned and non-empty")
            if s.lane_offset < prev_end:
                raise LayoutError(f"segment {s} overlaps its predecessor")
            prev_end = s.lane_offset + s.count
        want = (self.n, self.h, self.w, self.words_per_pixel)
        if words.shape != want:
            raise ShapeError(f"words shape {words.shape} != {want}")

    @property
    def lanes_per_pixel(self) -> int:
        return _round_block(max((s.lane_offset + s.count for s in self.segments), default=0))

    @property
    def words_per_pixel(self) -> int:
        return self.lanes_per_pixel // WORD_BITS

    @property
    def blocks_per_pixel(self) -> int:
        return self.lanes_per_pixel // BLOCK_BITS

    def lane_table(self) -> np.ndarray:
        return segment_lane_table(self.segments)

    def valid_lane_words(self) -> np.ndarray:
        bits = np.zeros(self.lanes_per_pixel, dtype=np.uint8)
        bits[self.lane_table()] = 1
        return bits_to_words(bits)

    def check_pad_lanes(self) -> None:
        if self.words.size and np.any(self.words & ~self.valid_lane_words()):
            raise LayoutError("pad lanes must be zero in every pixel")


def segment_lane_table(segments) -> np.ndarray:
    """Lane index of every logical channel (``layers.py:141-144``)."""
    if not segments:
        return np.zeros(0, dtype=np.int64)
    return np.concatenate(
        [s.lane_offset + np.arange(s.count, dtype=np.int64) for s in segments]
    )


def segment_lanes(segments) -> int:
    """Block-rounded per-pixel lane span of a layout (``layers.py:135-138``)."""
    return _round_block(max((s.lane_offset + s.count for s in segments), default=0))


def pack_bits_tensor(bits: np.ndarray) -> BitTensor:
    """bool (n, h, w, c) -> BitTensor, True = +1 (``bitcore.py:410-425``)."""
    b = np.asarray(bits, dtype=np.uint8)
    if b.ndim != 4:
        raise ShapeError(f"expected (n, h, w, c), got shape {b.shape}")
    n, h, w, c = b.shape
    if c == 0:
        return BitTensor(n, h, w, 0, np.zeros((n, h, w, 0), dtype=np.uint64), ())
    lanes = _round_block(c)
    full = np.zeros((n, h, w, lanes), dtype=np.uint8)
    full[..., :c] = b
    return BitTensor(n, h, w, c, bits_to_words(full), (ChannelSegment(0, c),))


def pack_tensor(values: np.ndarray) -> BitTensor:
    """{-1,+1} (n, h, w, c) -> BitTensor (``bitcore.py:391-407``)."""
    v = np.asarray(values)
    if v.ndim != 4:
        raise ShapeError(f"expected (n, h, w, c), got shape {v.shape}")
    if v.size and not np.isin(v, (-1, 1)).all():
        raise ValueAlphabetError("pack_tensor expects values in {-1,+1}")
    return pack_bits_tensor(v > 0)


def unpack_tensor(t) -> np.ndarray:
    """BitTensor -> int8 (n, h, w, c) of {-1,+1} (``bitcore.py:428-434``)."""
    if t.c == 0:
        return np.zeros((t.n, t.h, t.w, 0), dtype=np.int8)
    bits = words_to_bits(t.words)[..., segment_lane_table(t.segments)]
    return 2 * bits.astype(np.int8) - 1
