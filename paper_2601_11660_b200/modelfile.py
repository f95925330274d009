"""MBUN compiled-model files and RTEN raw tensors (host side, byte-compatible
with the reference's ``bitunet.modelfile``, ``pkg/src/bitunet/modelfile.py``).

This is the on-disk weight / mask format of SURVEY.md §8(f) rank 1: a model
trained and compiled elsewhere is read here and runs on the GPU unchanged
(``forward(read_model(path), image, device=...)`` or ``Engine``). Both
formats are little-endian; a written model re-reads to an identical
``CompiledModel`` and our writer emits the reference's bytes exactly
(pinned by ``tests/golden/*.mbun``, written by the reference itself).

Layouts (modelfile.py:1-38 of the reference):

``MBUN``: magic, u32 version 1; config (u32 height, width, in, out, stem,
encoder[4], tconv[4], decoder[4]; u16 precision id; u8 pad convention
(0 = out-of-bounds reads -1, 1 = zero padding); u8 sign(0) = +1 (always 1);
u8 stem2_float; u8 0); u32 layer count; per layer: u16 name length + name,
u8 kind code, u32 kh, kw, stride, padding, c_in, c_out (zeros for
maxpool / concat), then the payload -- float conv: u8 flags (1 bias,
2 batchnorm, 4 sign), f64 weights (c_out, kh, kw, c_in), f64 bias, f64
gamma / beta / mean / var and f64 eps; bit convs: u64 lane count + words of
the pos plane (masked kinds: then the neg plane), then c_out (i32 T, u8 code)
records; concat: the source layer name.

``RTEN``: magic, u32 version 1, u8 dtype (0 f32, 1 f64, 2 i32, 3 bit-packed),
u8 rank, u16 0, u64 extents, row-major payload (bit-packed: (n, h, w, c)
extents and the words of a single-segment ``BitTensor``).

Every parse failure raises ``FormatError`` with the byte offset.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .bitcore import BitPlane, BitTensor, MaskedWeightPlanes
from .errors import EngineError, FormatError
from .graph import CompiledLayer, CompiledModel, PrecisionMap, UNetConfig
from .layers import ConvSpec, FusedThreshold

__all__ = ["KIND_CODES", "read_model", "write_model", "read_tensor", "write_tensor"]

MODEL_MAGIC, TENSOR_MAGIC, VERSION = b"MBUN", b"RTEN", 1
KIND_CODES = {"float-conv": 0, "binary-conv": 1, "masked-conv": 2, "binary-tconv": 3,
              "masked-tconv": 4, "maxpool": 5, "concat": 6}
_KINDS = {code: kind for kind, code in KIND_CODES.items()}
BIAS, BATCHNORM, SIGN = 1, 2, 4
_RECORD = np.dtype([("t", "<i4"), ("code", "u1")])  # one threshold record, 5 bytes
_ARRAY_CODES = {np.dtype(np.float32): 0, np.dtype(np.float64): 1, np.dtype(np.int32): 2}
_ARRAY_TYPES = {code: dt.newbyteorder("<") for dt, code in _ARRAY_CODES.items()}
_CONFIG = struct.Struct("<5I4I4I4IH4B")


class _Cursor:
    """Bounds-checked little-endian reads over an in-memory file."""

    def __init__(self, blob: bytes, label: str):
        self.blob, self.pos, self.label = blob, 0, label

    def error(self, why: str) -> FormatError:
        return FormatError(f"{self.label}: {why}", where=f"byte {self.pos}")

    def bytes(self, n: int) -> bytes:
        end = self.pos + n
        if n < 0 or end > len(self.blob):
            raise self.error(f"truncated: wanted {n} bytes, {len(self.blob) - self.pos} left")
        chunk, self.pos = self.blob[self.pos:end], end
        return chunk

    def fields(self, layout: str | struct.Struct):
        s = layout if isinstance(layout, struct.Struct) else struct.Struct("<" + layout)
        return s.unpack(self.bytes(s.size))

    def one(self, code: str):
        return self.fields(code)[0]

    def values(self, dtype, count: int) -> np.ndarray:
        dt = np.dtype(dtype)
        return np.frombuffer(self.bytes(dt.itemsize * int(count)), dtype=dt).copy()

    def text(self) -> str:
        return self.bytes(self.one("H")).decode("utf-8")


def _text(name: str) -> bytes:
    raw = name.encode("utf-8")
    return struct.pack("<H", len(raw)) + raw


def _plane(plane: BitPlane) -> bytes:
    return struct.pack("<Q", plane.n_bits) + np.asarray(plane.words, dtype="<u8").tobytes()


def _records(th: FusedThreshold) -> bytes:
    rec = np.zeros(len(th.thresholds), dtype=_RECORD)
    rec["t"], rec["code"] = th.thresholds, th.codes
    return rec.tobytes()


def _f64(a) -> bytes:
    return np.ascontiguousarray(a, dtype="<f8").tobytes()


def write_model(model: CompiledModel, path) -> None:
    """Serialize a ``CompiledModel`` (reference ``write_model``, modelfile.py:124-170)."""
    c = model.config
    parts = [MODEL_MAGIC, struct.pack("<I", VERSION),
             _CONFIG.pack(c.height, c.width, c.in_channels, c.out_channels, c.stem_channels,
                          *c.encoder_channels, *c.tconv_channels, *c.decoder_channels,
                          c.precision.config_id(), int(c.pad_mode == "zero"), 1,
                          int(bool(c.stem2_float)), 0),
             struct.pack("<I", len(model.layers))]
    for layer in model.layers:
        s = layer.spec
        geom = (0,) * 6 if s is None else (s.kernel_h, s.kernel_w, s.stride, s.padding,
                                            s.c_in, s.c_out)
        parts += [_text(layer.name), struct.pack("<B6I", KIND_CODES[layer.kind], *geom)]
        kind = layer.kind
        if kind == "float-conv":
            flags = ((BIAS if layer.bias is not None else 0) | (BATCHNORM if layer.bn is not None else 0)
                     | (SIGN if layer.apply_sign else 0))
            parts += [struct.pack("<B", flags), _f64(layer.weights)]
            if layer.bias is not None:
                parts.append(_f64(layer.bias))
            if layer.bn is not None:
                *arrays, eps = layer.bn
                parts += [_f64(a) for a in arrays] + [struct.pack("<d", eps)]
        elif kind.startswith("binary-"):
            parts += [_plane(layer.weights), _records(layer.threshold)]
        elif kind.startswith("masked-"):
            parts += [_plane(layer.weights.pos), _plane(layer.weights.neg), _records(layer.threshold)]
        elif kind == "concat":
            parts.append(_text(layer.concat_with))
    Path(path).write_bytes(b"".join(parts))


def _read_plane(cur: _Cursor) -> BitPlane:
    n_bits = cur.one("Q")
    return BitPlane(int(n_bits), cur.values("<u8", -(-n_bits // 64)).astype(np.uint64))


def _read_layer(cur: _Cursor, pad_mode: str) -> CompiledLayer:
    name = cur.text()
    code = cur.one("B")
    if code not in _KINDS:
        raise cur.error(f"unknown layer kind code {code}")
    kind = _KINDS[code]
    kh, kw, stride, padding, c_in, c_out = cur.fields("6I")
    try:
        spec = None
        if kind not in ("maxpool", "concat"):
            # only the bit convs carry the model's padding convention
            spec = ConvSpec(kh, kw, stride, padding, c_in, c_out,
                            pad_mode=pad_mode if kind.endswith("-conv") and kind != "float-conv"
                            else "neg_one")
        if kind == "float-conv":
            flags = cur.one("B")
            w = cur.values("<f8", c_out * kh * kw * c_in).reshape(c_out, kh, kw, c_in)
            bias = cur.values("<f8", c_out) if flags & BIAS else None
            bn = None
            if flags & BATCHNORM:
                arrays = [cur.values("<f8", c_out) for _ in range(4)]
                bn = (*arrays, cur.one("d"))
            return CompiledLayer(name, kind, spec, weights=w, bias=bias, bn=bn,
                                 apply_sign=bool(flags & SIGN))
        if kind in ("maxpool", "concat"):
            return CompiledLayer(name, kind, concat_with=cur.text() if kind == "concat" else "")
        if kind.startswith("masked-"):
            weights = MaskedWeightPlanes(_read_plane(cur), _read_plane(cur))
        else:
            weights = _read_plane(cur)
        rec = cur.values(_RECORD, c_out)
        return CompiledLayer(name, kind, spec, weights=weights,
                             threshold=FusedThreshold(rec["t"], rec["code"]))
    except FormatError:
        raise
    except EngineError as exc:
        raise cur.error(f"layer {name!r} is inconsistent: {exc}") from exc


def read_model(path) -> CompiledModel:
    """Parse an MBUN file (reference ``read_model``, modelfile.py:179-289)."""
    cur = _Cursor(Path(path).read_bytes(), f"model file {path}")
    if cur.bytes(4) != MODEL_MAGIC:
        cur.pos = 0
        raise cur.error("bad magic (expected MBUN)")
    version = cur.one("I")
    if version != VERSION:
        raise cur.error(f"unsupported version {version}")
    f = cur.fields(_CONFIG)
    (height, width, in_c, out_c, stem_c), enc, tcv, dec = f[:5], f[5:9], f[9:13], f[13:17]
    precision_id, pad_flag, sign_flag, stem2_float, _ = f[17:]
    if precision_id >= 4096:
        raise cur.error(f"precision id {precision_id} has nonzero top bits")
    if pad_flag > 1 or sign_flag != 1:
        raise cur.error(f"unknown convention flags pad={pad_flag} sign={sign_flag}")
    pad_mode = "zero" if pad_flag else "neg_one"
    try:
        config = UNetConfig(in_channels=in_c, height=height, width=width, stem_channels=stem_c,
                            encoder_channels=enc, tconv_channels=tcv, decoder_channels=dec,
                            out_channels=out_c, precision=PrecisionMap.from_config_id(precision_id),
                            stem2_float=bool(stem2_float), pad_mode=pad_mode)
    except EngineError as exc:
        raise cur.error(f"bad config block: {exc}") from exc
    layers = tuple(_read_layer(cur, pad_mode) for _ in range(cur.one("I")))
    if cur.pos != len(cur.blob):
        raise cur.error(f"{len(cur.blob) - cur.pos} trailing bytes")
    return CompiledModel(config, layers)


def write_tensor(path, value) -> None:
    """Serialize an f32 / f64 / i32 array or a single-segment ``BitTensor``."""
    head = [TENSOR_MAGIC, struct.pack("<I", VERSION)]
    if isinstance(value, BitTensor):
        if len(value.segments) > 1:
            raise FormatError("only single-segment bit tensors are serializable")
        body = [struct.pack("<BBH4Q", 3, 4, 0, value.n, value.h, value.w, value.c),
                np.asarray(value.words, dtype="<u8").tobytes()]
    else:
        arr = np.asarray(value)
        if arr.dtype not in _ARRAY_CODES:
            raise FormatError(f"unsupported tensor dtype {arr.dtype}")
        body = [struct.pack(f"<BBH{arr.ndim}Q", _ARRAY_CODES[arr.dtype], arr.ndim, 0, *arr.shape),
                np.ascontiguousarray(arr, dtype=arr.dtype.newbyteorder("<")).tobytes()]
    Path(path).write_bytes(b"".join(head + body))


def read_tensor(path):
    """Parse an RTEN file: an ndarray, or a ``BitTensor`` for dtype 3."""
    cur = _Cursor(Path(path).read_bytes(), f"tensor file {path}")
    if cur.bytes(4) != TENSOR_MAGIC:
        cur.pos = 0
        raise cur.error("bad magic (expected RTEN)")
    version = cur.one("I")
    if version != VERSION:
        raise cur.error(f"unsupported version {version}")
    code, rank, _ = cur.fields("BBH")
    shape = cur.fields(f"{rank}Q")
    if code == 3:
        if rank != 4:
            raise cur.error(f"bit-packed tensors have rank 4, got {rank}")
        n, h, w, c = (int(e) for e in shape)
        wpp = -(-c // 128) * 2
        words = cur.values("<u8", n * h * w * wpp).astype(np.uint64).reshape(n, h, w, wpp)
        try:
            out = BitTensor(n, h, w, c, words)
            out.check_pad_lanes()
        except EngineError as exc:
            raise cur.error(str(exc)) from exc
    elif code in _ARRAY_TYPES:
        dt = _ARRAY_TYPES[code]
        out = cur.values(dt, int(np.prod(shape, dtype=np.int64))).reshape(shape).astype(dt.newbyteorder("="))
    else:
        raise cur.error(f"unknown dtype code {code}")
    if cur.pos != len(cur.blob):
        raise cur.error(f"{len(cur.blob) - cur.pos} trailing bytes")
    return out
