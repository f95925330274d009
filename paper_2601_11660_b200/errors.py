"""Exception taxonomy of the engine, mirroring ``bitunet.errors``.

Reference: ``pkg/src/bitunet/errors.py:8-44``. The class names, the
hierarchy and the ``where`` attribute of :class:`FormatError` are identical.
When the reference package itself is importable, every class here also
SUBCLASSES its ``bitunet.errors`` namesake, so ``except
bitunet.errors.ShapeError`` catches the engine's errors unchanged (the
drop-in contract; ``MBU_REFERENCE_ERRORS=0`` turns that off). Without
``bitunet`` (e.g. on a serving box) the classes stand alone.

The C-ABI (``include/mbunet.h``) never lets an exception cross the library
boundary: every entry point returns an ``int`` status. :data:`STATUS_CLASSES`
maps those codes back onto the Python classes, and :func:`raise_for_status`
is what the ctypes wrapper calls after every C call.
"""

from __future__ import annotations

import importlib.util
import os


def _reference_errors():
    if os.environ.get("MBU_REFERENCE_ERRORS", "1") == "0":
        return None
    try:
        if importlib.util.find_spec("bitunet") is None:
            return None
        import bitunet.errors as ref

        return ref
    except Exception:  # noqa: BLE001 - a broken reference install only disables the aliasing
        return None


_REF = _reference_errors()


def _also(name: str) -> tuple:
    """The reference's class of that name, as an extra base (or nothing)."""
    cls = getattr(_REF, name, None) if _REF is not None else None
    return (cls,) if isinstance(cls, type) else ()


class EngineError(*_also("EngineError"), Exception):
    """Root of every engine-raised error (``errors.py:8``)."""


class ValueAlphabetError(EngineError, *_also("ValueAlphabetError")):
    """A value lies outside its alphabet ({-1,+1} or {-1,0,+1})."""


class LayoutError(EngineError, *_also("LayoutError")):
    """Lane / word / plane layouts disagree."""


class PlaneOverlapError(EngineError, *_also("PlaneOverlapError")):
    """A weight lane is set in both the pos and the neg plane."""


class ShapeError(EngineError, *_also("ShapeError")):
    """Tensor extents do not fit the requested operation."""


class UnsupportedConfigError(EngineError, *_also("UnsupportedConfigError")):
    """A configuration the engine deliberately does not express."""


class FormatError(EngineError, *_also("FormatError")):
    """A file failed to parse; ``where`` locates the problem."""

    def __init__(self, message, where=None):
        if where is not None:
            message = f"{message} (at {where})"
        Exception.__init__(self, message)  # (not the reference's __init__: it would re-append)
        self.where = where


class BundleError(FormatError, *_also("BundleError")):
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
