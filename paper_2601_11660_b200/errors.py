"""Exception taxonomy of the engine, mirroring ``bitunet.errors``.

Reference: ``pkg/src/bitunet/errors.py:8-44``. The class names, the
hierarchy and the ``where`` attribute of :class:`FormatError` are identical,
so callers that catch the reference's exceptions catch ours unchanged.

The C-ABI (``include/mbunet.h``) never lets an exception cross the library
boundary: every entry point returns an ``int`` status. :data:`STATUS_CLASSES`
maps those codes back onto the Python classes, and :func:`raise_for_status`
is what the ctypes wrapper calls after every C call.
"""

from __future__ import annotations


class EngineError(Exception):
    """Root of every engine-raised error (``errors.py:8``)."""


class ValueAlphabetError(EngineError):
    """A value lies outside its alphabet ({-1,+1} or {-1,0,+1})."""


class LayoutError(EngineError):
    """Lane / word / plane layouts disagree."""


class PlaneOverlapError(EngineError):
    """A weight lane is set in both the pos and the neg plane."""


class ShapeError(EngineError):
    """Tensor extents do not fit the requested operation."""


class UnsupportedConfigError(EngineError):
    """A configuration the engine deliberately does not express."""


class FormatError(EngineError):
    """A file failed to parse; ``where`` locates the problem."""

    def __init__(self, message, where=None):
        self.where = where
        if where is not None:
            message = f"{message} (at {where})"
        super().__init__(message)


class BundleError(FormatError):
    """A weight bundle directory or manifest is malformed."""


class CudaError(EngineError):
    """A CUDA runtime / launch failure reported by ``libmbunet``."""


# Status codes returned by every ``mbu_*`` C entry point (include/mbunet.h).
MBU_OK = 0
STATUS_CLASSES = {
    1: EngineError,
    2: ValueAlphabetError,
    3: LayoutError,
    4: PlaneOverlapError,
    5: ShapeError,
    6: UnsupportedConfigError,
    7: CudaError,
}


def raise_for_status(status: int, message: str) -> None:
    """Raise the Python class that corresponds to a C status code."""
    if status == MBU_OK:
        return
    cls = STATUS_CLASSES.get(int(status), EngineError)
    raise cls(message or f"libmbunet status {status}")
