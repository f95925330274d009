"""Compile the oracle's C restatement for the current host — TEST INFRA ONLY.

The library is keyed by the host CPU (``-march=native``), because the
build container and the GPU box may have different CPUs; gcc is present on
both. Output goes to ``oracle/_build/`` (git-ignored).
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import platform
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent


def _cpu_key() -> str:
    try:
        flags = next(l for l in open("/proc/cpuinfo") if l.startswith("flags"))
    except (OSError, StopIteration):
        flags = platform.processor()
    return hashlib.sha1(flags.encode()).hexdigest()[:12]


def lib_path() -> Path:
    return HERE / "_build" / _cpu_key() / "liboracle_xorpop.so"


def build(force: bool = False) -> Path:
    out = lib_path()
    src = HERE / "xorpop.c"
    if out.exists() and not force and out.stat().st_mtime >= src.stat().st_mtime:
        return out
    out.parent.mkdir(parents=True, exist_ok=True)
    tmp = out.with_suffix(f".{os.getpid()}.tmp")
    subprocess.run(
        ["gcc", "-O3", "-march=native", "-fopenmp", "-shared", "-fPIC", str(src), "-o", str(tmp)],
        check=True,
    )
    os.replace(tmp, out)
    return out


_LIB = None


def load():
    global _LIB
    if _LIB is None:
        lib = ctypes.CDLL(str(build()))
        fn = lib.oracle_xor_popcount_rows
        fn.restype = None
        fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                       ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int]
        _LIB = lib
    return _LIB
