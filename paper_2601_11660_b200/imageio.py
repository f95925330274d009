"""Netpbm image input (P5 / P6) and mask output, byte-compatible with the
reference's ``bitunet.imageio`` (``pkg/src/bitunet/imageio.py``).

``read_image`` returns what the reference's does: float64 (1, h, w, c) with
values ``sample / maxval``. For frame streams the decode belongs on the GPU
(SURVEY.md §8(f) rank 2): ``read_raster`` hands back the undecoded samples
(u8, or big-endian u16 as raw bytes) and ``decode_raster`` turns them into
the float64 image on the device with the same correctly rounded division
(``mbu_decode_raster``), so only 1-2 bytes per sample cross PCIe instead of 8.
Malformed headers raise ``FormatError`` with the byte offset.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

from .errors import FormatError, ShapeError

__all__ = ["read_image", "read_raster", "write_mask", "write_gray"]

_SPACE = frozenset(b for b in range(256) if chr(b).isspace())  # the reference tests chr().isspace()


def _header(data: bytes, label: str):
    """Parse ``magic width height maxval`` (comments allowed); returns the fields
    and the raster offset (one whitespace byte after maxval, imageio.py:75)."""
    pos, tokens = 0, []
    while len(tokens) < 4:
        while pos < len(data) and (data[pos] in _SPACE or data[pos] == 0x23):
            if data[pos] == 0x23:  # '#' comment to end of line
                while pos < len(data) and data[pos] not in b"\r\n":
                    pos += 1
            else:
                pos += 1
        if pos >= len(data):
            raise FormatError(f"{label}: truncated header", where=f"byte {pos}")
        start = pos
        while pos < len(data) and data[pos] not in _SPACE and data[pos] != 0x23:
            pos += 1
        tok = data[start:pos]
        if not tokens:
            if tok not in (b"P5", b"P6"):
                raise FormatError(f"{label}: unsupported magic {tok!r} (want P5 or P6)", where="byte 0")
        else:
            name = ("width", "height", "maxval")[len(tokens) - 1]
            try:
                value = int(tok.decode("ascii"), 10)
            except (UnicodeDecodeError, ValueError) as exc:
                raise FormatError(f"{label}: {name}: {tok!r} is not a decimal integer",
                                  where=f"byte {pos}") from exc
            if value <= 0:
                raise FormatError(f"{label}: {name} must be positive, got {value}", where=f"byte {pos}")
            tok = value
        tokens.append(tok)
    magic, width, height, maxval = tokens
    if maxval > 65535:
        raise FormatError(f"{label}: maxval {maxval} exceeds 65535", where=f"byte {pos}")
    return magic, width, height, maxval, pos + 1


def read_raster(path):
    """Undecoded samples of a P5/P6 file: (raster uint8 array of shape
    (1, h, w, c) for maxval <= 255, else (1, h, w, c, 2) big-endian byte
    pairs), maxval."""
    data = Path(path).read_bytes()
    label = f"image file {path}"
    magic, width, height, maxval, off = _header(data, label)
    c = 1 if magic == b"P5" else 3
    bps = 2 if maxval > 255 else 1
    need = width * height * c * bps
    raster = data[off:off + need]
    if len(raster) != need:
        raise FormatError(f"{label}: raster truncated: wanted {need} bytes, got {len(raster)}",
                          where=f"byte {off}")
    shape = (1, height, width, c) + ((2,) if bps == 2 else ())
    return np.frombuffer(raster, dtype=np.uint8).reshape(shape).copy(), maxval


def read_image(path) -> np.ndarray:
    """float64 (1, h, w, c) in [0, 1], decoded on the host (imageio.py:59-83)."""
    raster, maxval = read_raster(path)
    if raster.ndim == 5:
        samples = raster[..., 0].astype(np.uint32) << 8 | raster[..., 1]
    else:
        samples = raster
    return samples.astype(np.float64) / maxval


def write_mask(path, mask: np.ndarray) -> None:
    """(h, w) or (1, h, w) {0, 1} -> P5 with values {0, 255}."""
    m = np.squeeze(np.asarray(mask))
    if m.ndim != 2:
        raise ShapeError(f"mask must be 2-d, got shape {np.asarray(mask).shape}")
    body = np.where(m != 0, 255, 0).astype(np.uint8).tobytes()
    Path(path).write_bytes(f"P5\n{m.shape[1]} {m.shape[0]}\n255\n".encode("ascii") + body)


def write_gray(path, image: np.ndarray) -> None:
    """[0, 1] floats (h, w) -> 8-bit P5, rounding half away from zero."""
    img = np.squeeze(np.asarray(image, dtype=np.float64))
    if img.ndim != 2:
        raise ShapeError(f"grayscale image must be 2-d, got shape {np.asarray(image).shape}")
    body = np.clip(np.floor(img * 255.0 + 0.5), 0, 255).astype(np.uint8).tobytes()
    Path(path).write_bytes(f"P5\n{img.shape[1]} {img.shape[0]}\n255\n".encode("ascii") + body)
