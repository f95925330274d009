"""ctypes binding of ``libmbunet.so`` (the C-ABI declared in include/mbunet.h).

The library is built in-tree by ``__graft_entry__.build()`` (plain nvcc,
``-gencode arch=compute_100a,code=sm_100a``). There is no fallback: if the
library is missing, or no CUDA device is present, every GPU entry point
raises — the product never silently computes on the CPU.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import EngineError, raise_for_status

LIB_PATH = Path(__file__).resolve().parent / "libmbunet.so"

MBU_PAD_NEG_ONE = 0
MBU_PAD_ZERO = 1
PATH_AUTO = 0
PATH_TCGEN05 = 1
PATH_POPCOUNT = 2

_c = ctypes
_vp = _c.c_void_p
_i = _c.c_int
_i64 = _c.c_int64
_sz = _c.c_size_t

_SIGS = {
    "mbu_last_error": (_c.c_char_p, []),
    "mbu_version": (_i, []),
    "mbu_launch_count": (_i64, []),
    "mbu_last_path": (_i, []),
    "mbu_set_option": (_i, [_i, _i]),
    "mbu_argmax": (_i, [_vp, _i64, _i, _vp, _vp]),
    "mbu_pack_mask": (_i, [_vp, _i64, _i64, _vp, _vp]),
    "mbu_decode_raster": (_i, [_vp, _i64, _i, _i, _vp, _vp]),
    "mbu_quantize_weights": (_i, [_vp, _i64, _i, _c.c_double, _vp, _vp]),
    "mbu_quantize_weights_f64": (_i, [_vp, _i64, _i, _c.c_double, _vp, _vp]),
    "mbu_fuse_bn_sign": (_i, [_vp, _vp, _vp, _vp, _c.c_double, _vp, _i, _vp, _vp, _vp]),
    "mbu_conv_create": (_i, [_c.POINTER(_vp), _i, _i, _i, _i, _i, _i, _i, _i, _i, _i,
                             _vp, _vp, _vp, _vp, _vp, _vp]),
    "mbu_conv_destroy": (_i, [_vp]),
    "mbu_conv_run": (_i, [_vp, _vp, _i, _i, _i, _i, _i, _vp, _vp, _i, _i, _i, _vp]),
    "mbu_threshold_pack": (_i, [_vp, _i64, _i, _vp, _vp, _vp, _i, _i, _vp]),
    "mbu_maxpool2": (_i, [_vp, _i, _i, _i, _i, _i, _i, _vp, _i, _i, _vp]),
    "mbu_xor_popcount_rows": (_i, [_vp, _vp, _vp, _i64, _i64, _i64, _vp]),
    "mbu_fconv_create": (_i, [_c.POINTER(_vp), _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp,
                              _c.c_double, _vp]),
    "mbu_fconv_destroy": (_i, [_vp]),
    "mbu_fconv_run": (_i, [_vp, _vp, _vp, _i, _i, _i, _i, _i, _vp, _vp, _i, _i, _vp, _vp]),
    "mbu_model_create": (_i, [_c.POINTER(_vp), _i]),
    "mbu_model_destroy": (_i, [_vp]),
    "mbu_model_add_conv": (_i, [_vp, _vp]),
    "mbu_model_add_fconv": (_i, [_vp, _vp, _i]),
    "mbu_model_add_maxpool": (_i, [_vp]),
    "mbu_model_add_concat": (_i, [_vp, _i]),
    "mbu_model_plan": (_i, [_vp, _i, _i, _i, _i, _c.POINTER(_sz)]),
    "mbu_forward": (_i, [_vp, _vp, _vp, _vp, _vp, _sz, _i, _vp]),
    "mbu_model_set_timing": (_i, [_vp, _i]),
    "mbu_model_layer_times": (_i, [_vp, _c.POINTER(_c.c_float)]),
    "mbu_model_layer_info": (_i, [_vp, _i] + [_c.POINTER(_i)] * 7
                             + [_c.POINTER(_sz), _c.POINTER(_sz), _c.POINTER(_i)]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(path: str | os.PathLike | None = None):
    """Load and type the library (no CUDA work happens here)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else Path(os.environ.get("MBU_LIB", LIB_PATH))
    if not p.exists():
        raise EngineError(
            f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if os.environ.get("MBU_CONV_I8"):  # A/B switch for benchmarks: 3x3 convs on kind::i8
        lib.mbu_set_option(3, 1)
    if os.environ.get("MBU_FUSED_HEAD"):  # A/B switch: the head in up-C4.b's epilogue
        lib.mbu_set_option(4, 1)
    if path is None:
        _lib = lib
    return lib


def call(name: str, *args) -> None:
    """Call ``name`` and raise the mapped EngineError subclass on failure."""
    lib = load()
    status = getattr(lib, name)(*args)
    if status:
        msg = lib.mbu_last_error()
        raise_for_status(status, msg.decode() if msg else "")


def launch_count() -> int:
    return int(load().mbu_launch_count())


def last_path() -> int:
    return int(load().mbu_last_path())
