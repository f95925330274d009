"""Layer-level operators of the reference API, executed on sm_100a.

Drop-in replacements for the data-parallel functions of
``pkg/src/bitunet/layers.py`` and ``bitcore.py``, same names, arguments,
return types and error behaviour:

=============================  ==========================================
reference (file:line)          here -> libmbunet entry point
=============================  ==========================================
conv_forward (layers.py:289)   conv_forward -> mbu_conv_create/_run
transposed_conv_forward (:316) transposed_conv_forward -> mbu_conv_run
apply_threshold (:508)         apply_threshold -> mbu_threshold_pack
maxpool2 (:360)                maxpool2 -> mbu_maxpool2
float_conv (:530)              float_conv -> mbu_fconv_run
float_bn_sign (:553)           float_bn_sign -> mbu_fconv_run (1x1 identity)
bit_gemm (bitcore.py:265)      bit_gemm -> mbu_xor_popcount_rows
xor_popcount_rows (kernels:114) xor_popcount_rows -> mbu_xor_popcount_rows
=============================  ==========================================

Host arrays in, host arrays out (the reference contract); each call moves
its operands to the GPU, runs there and copies the result back. ``threads``
is accepted and ignored (results never depend on it, as in the reference).
The whole-network path (:mod:`.runtime`) keeps everything resident instead.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .bitcore import BitTensor, ChannelSegment, PackedBitMatrix, is_masked, segment_lanes
from .errors import EngineError, LayoutError, PlaneOverlapError, ShapeError, UnsupportedConfigError
from .layers import ConvSpec, FusedThreshold

__all__ = [
    "cuda_device",
    "ConvHandle",
    "FloatConvHandle",
    "conv_forward",
    "transposed_conv_forward",
    "apply_threshold",
    "maxpool2",
    "float_conv",
    "float_bn_sign",
    "bit_gemm",
    "xor_popcount_rows",
    "quantize_weights",
    "fuse_bn_sign",
]


def cuda_device(device=None) -> torch.device:
    """The CUDA device to run on; raises if there is none (no CPU fallback)."""
    if not torch.cuda.is_available():
        raise EngineError("no CUDA device: the MBU-Net engine runs only on sm_100a GPUs")
    d = torch.device("cuda") if device is None else torch.device(device)
    if d.type != "cuda":
        raise EngineError(f"device {d} is not a CUDA device")
    if d.index is None:
        d = torch.device("cuda", torch.cuda.current_device())
    return d


def _ptr(t) -> ctypes.c_void_p:
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data_as(ctypes.c_void_p)
    return ctypes.c_void_p(t.data_ptr())


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _words_to_dev(words: np.ndarray, device) -> torch.Tensor:
    w = np.ascontiguousarray(words, dtype=np.uint64)
    return torch.from_numpy(w.view(np.int64)).to(device)


def _dev_to_words(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


class ConvHandle:
    """Uploaded, repacked weights of one bit conv / transposed conv.

    Validation mirrors the reference before any device work:
    ``UnsupportedConfigError`` for binary + zero padding (``layers.py:296-299``)
    and for tconvs with kernel != stride or padding (``layers.py:320-326``),
    ``LayoutError`` for plane sizes (``layers.py:222-225``),
    ``PlaneOverlapError`` for pos & neg (``bitcore.py:285-286``).
    """

    def __init__(self, weights, spec: ConvSpec, segments, threshold=None, transposed=False,
                 device=None):
        self.device = cuda_device(device)
        self.spec = spec
        self.transposed = bool(transposed)
        masked = is_masked(weights)
        if spec.pad_mode == "zero" and not masked and not transposed:
            raise UnsupportedConfigError(
                "binary convs cannot zero-pad: {-1,+1} activations have no 0 state")
        if transposed:
            if spec.kernel_h != spec.stride or spec.kernel_w != spec.stride:
                raise UnsupportedConfigError(
                    f"transposed conv requires kernel = stride, got {spec.kernel_h}x{spec.kernel_w}"
                    f" stride {spec.stride}")
            if spec.padding:
                raise UnsupportedConfigError("transposed conv does not support padding")
        first = weights.pos if masked else weights
        lpp = segment_lanes(segments)
        k_lanes = spec.kernel_h * spec.kernel_w * lpp
        if not hasattr(first, "n_bits") or first.n_bits != spec.c_out * k_lanes:
            raise LayoutError(
                f"weight plane has {getattr(first, 'n_bits', None)} lanes, expected "
                f"{spec.c_out}*{k_lanes}")
        pos = np.ascontiguousarray(first.words, dtype=np.uint64)
        neg = np.ascontiguousarray(weights.neg.words, dtype=np.uint64) if masked else None
        if neg is not None and np.any(pos & neg):
            raise PlaneOverlapError("a weight lane is set in both pos and neg planes")
        offs = np.array([s.lane_offset for s in segments], dtype=np.int32)
        cnts = np.array([s.count for s in segments], dtype=np.int32)
        thr = codes = None
        if threshold is not None:
            thr = np.ascontiguousarray(threshold.thresholds, dtype=np.int32)
            codes = np.ascontiguousarray(threshold.codes, dtype=np.uint8)
            if thr.shape != (spec.c_out,):
                raise ShapeError(f"{thr.shape[0]} thresholds for {spec.c_out} channels")
        self.wpp = lpp // 64
        self.out_wpp = ((spec.c_out + 127) // 128) * 2
        self.segments = tuple(segments)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.call("mbu_conv_create", ctypes.byref(h), self.device.index, int(transposed),
                      spec.kernel_h, spec.kernel_w, spec.stride, spec.padding, spec.c_in,
                      spec.c_out, _lib.MBU_PAD_ZERO if spec.pad_mode == "zero" and not transposed else 0,
                      len(segments), _ptr(offs), _ptr(cnts), _ptr(pos), _ptr(neg), _ptr(thr),
                      _ptr(codes))
        self.handle = h
        self._owned = True

    def out_extent(self, h, w):
        if self.transposed:
            return h * self.spec.stride, w * self.spec.stride
        return self.spec.out_extent(h, w)

    def run(self, x_dev: torch.Tensor, n, h, w, x_stride=None, x_offset=0, acc=None, bits=None,
            out_stride=None, out_offset=0, path=_lib.PATH_AUTO):
        """Device-level call: x_dev / acc / bits are CUDA tensors."""
        _lib.call("mbu_conv_run", self.handle, _ptr(x_dev), n, h, w,
                  self.wpp if x_stride is None else x_stride, x_offset, _ptr(acc), _ptr(bits),
                  self.out_wpp if out_stride is None else out_stride, out_offset, path,
                  _stream(self.device))

    def release(self):
        """Hand ownership to a model (mbu_model_add_conv)."""
        self._owned = False
        return self.handle

    def __del__(self):
        if getattr(self, "_owned", False) and _lib._lib is not None:
            _lib.load().mbu_conv_destroy(self.handle)
            self._owned = False


class FloatConvHandle:
    """Uploaded float64 endpoint conv (stem / stem2_float / head)."""

    def __init__(self, weights, bias, spec: ConvSpec, bn=None, in_lanes=None, device=None):
        self.device = cuda_device(device)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        if w.shape != (spec.c_out, spec.kernel_h, spec.kernel_w, spec.c_in):
            raise ShapeError(f"weight shape {w.shape} inconsistent with {spec}")
        b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float64).reshape(-1)
        bnv = eps = None
        if bn is not None:
            gamma, beta, mean, var, eps = bn
            bnv = np.ascontiguousarray(np.concatenate([
                np.asarray(v, dtype=np.float64).reshape(-1) for v in (gamma, beta, mean, var)]))
        lanes = None if in_lanes is None else np.ascontiguousarray(in_lanes, dtype=np.int32)
        self.spec = spec
        self.out_wpp = ((spec.c_out + 127) // 128) * 2
        self.bits_input = lanes is not None
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.call("mbu_fconv_create", ctypes.byref(h), self.device.index, spec.kernel_h,
                      spec.kernel_w, spec.stride, spec.padding, spec.c_in, spec.c_out, _ptr(w),
                      _ptr(b), _ptr(bnv), float(eps or 0.0), _ptr(lanes))
        self.handle = h
        self._owned = True

    def run(self, n, h, w, x_f64=None, x_bits=None, x_stride=0, x_offset=0, acc=None, bits=None,
            mask=None):
        _lib.call("mbu_fconv_run", self.handle, _ptr(x_f64), _ptr(x_bits), x_stride, x_offset,
                  n, h, w, _ptr(acc), _ptr(bits), self.out_wpp, 0, _ptr(mask),
                  _stream(self.device))

    def release(self):
        self._owned = False
        return self.handle

    def __del__(self):
        if getattr(self, "_owned", False) and _lib._lib is not None:
            _lib.load().mbu_fconv_destroy(self.handle)
            self._owned = False


# --------------------------------------------------------------------------- #
# reference-shaped layer API (host arrays in / out)
# --------------------------------------------------------------------------- #


def _bit_layer(x, weights, spec, transposed, path, device):
    if spec.c_in != x.c:
        raise ShapeError(f"spec c_in {spec.c_in} != input channels {x.c}")
    conv = ConvHandle(weights, spec, x.segments, None, transposed=transposed, device=device)
    ho, wo = conv.out_extent(x.h, x.w)
    dev = conv.device
    xd = _words_to_dev(x.words, dev)
    acc = torch.empty((x.n, ho, wo, spec.c_out), dtype=torch.int32, device=dev)
    conv.run(xd, x.n, x.h, x.w, acc=acc, path=path)
    return acc.cpu().numpy()


def conv_forward(x, weights, spec: ConvSpec, threads: int = 1, *, path=_lib.PATH_AUTO,
                 device=None) -> np.ndarray:
    """Exact int32 conv of a packed tensor (``layers.py:289-313``), on the GPU."""
    return _bit_layer(x, weights, spec, False, path, device)


def transposed_conv_forward(x, weights, spec: ConvSpec, threads: int = 1, *,
                            path=_lib.PATH_AUTO, device=None) -> np.ndarray:
    """Kernel == stride transposed conv (``layers.py:316-352``), on the GPU."""
    return _bit_layer(x, weights, spec, True, path, device)


def apply_threshold(acc, t, *, device=None) -> BitTensor:
    """int32 accumulators vs fused thresholds -> packed bits (``layers.py:508-522``)."""
    acc = np.asarray(acc)
    if acc.ndim != 4:
        raise ShapeError(f"expected (n, h, w, c) accumulators, got {acc.shape}")
    if acc.shape[-1] != t.n_channels:
        raise ShapeError(f"{acc.shape[-1]} channels vs {t.n_channels} threshold entries")
    dev = cuda_device(device)
    n, h, w, c = acc.shape
    if c == 0:
        return BitTensor(n, h, w, 0, np.zeros((n, h, w, 0), dtype=np.uint64), ())
    wpp = ((c + 127) // 128) * 2
    ad = torch.from_numpy(np.ascontiguousarray(acc, dtype=np.int32)).to(dev)
    td = torch.from_numpy(np.ascontiguousarray(t.thresholds, dtype=np.int32)).to(dev)
    cd = torch.from_numpy(np.ascontiguousarray(t.codes, dtype=np.uint8)).to(dev)
    out = torch.empty((n, h, w, wpp), dtype=torch.int64, device=dev)
    _lib.call("mbu_threshold_pack", _ptr(ad), n * h * w, c, _ptr(td), _ptr(cd), _ptr(out), wpp,
              0, _stream(dev))
    return BitTensor(n, h, w, c, _dev_to_words(out), (ChannelSegment(0, c),))


def maxpool2(x, *, device=None) -> BitTensor:
    """2x2 max-pool as a wordwise OR (``layers.py:360-366``)."""
    if x.h % 2 or x.w % 2:
        raise ShapeError(f"extents must be even, got {x.h}x{x.w}")
    dev = cuda_device(device)
    wpp = x.words_per_pixel
    ho, wo = x.h // 2, x.w // 2
    if wpp == 0 or x.n * ho * wo == 0:
        return BitTensor(x.n, ho, wo, x.c, np.zeros((x.n, ho, wo, wpp), dtype=np.uint64),
                         x.segments)
    xd = _words_to_dev(x.words, dev)
    out = torch.empty((x.n, ho, wo, wpp), dtype=torch.int64, device=dev)
    _lib.call("mbu_maxpool2", _ptr(xd), x.n, x.h, x.w, wpp, wpp, 0, _ptr(out), wpp, 0,
              _stream(dev))
    return BitTensor(x.n, ho, wo, x.c, _dev_to_words(out), x.segments)


def float_conv(x, w, bias, spec: ConvSpec, *, device=None) -> np.ndarray:
    """float64 conv with zero padding (``layers.py:530-550``), on the GPU."""
    x = np.asarray(x, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    if x.ndim != 4 or w.ndim != 4:
        raise ShapeError(f"expected 4-d activations/weights, got {x.shape} / {w.shape}")
    n, h, wd, ci = x.shape
    if w.shape != (spec.c_out, spec.kernel_h, spec.kernel_w, spec.c_in) or ci != spec.c_in:
        raise ShapeError(f"weight shape {w.shape} inconsistent with {spec}")
    ho, wo = spec.out_extent(h, wd)
    fc = FloatConvHandle(w, bias, spec, device=device)
    xd = torch.from_numpy(np.ascontiguousarray(x)).to(fc.device)
    out = torch.empty((n, ho, wo, spec.c_out), dtype=torch.float64, device=fc.device)
    fc.run(n, h, wd, x_f64=xd, acc=out)
    return out.cpu().numpy()


def float_bn_sign(acc, gamma, beta, mean, var, eps, bias=None, *, device=None) -> BitTensor:
    """BN + sign + pack on float accumulators (``layers.py:553-560``)."""
    acc = np.asarray(acc, dtype=np.float64)
    n, h, w, c = acc.shape
    ident = np.eye(c, dtype=np.float64).reshape(c, 1, 1, c)
    spec = ConvSpec(1, 1, 1, 0, c, c)
    fc = FloatConvHandle(ident, bias, spec, bn=(gamma, beta, mean, var, eps), device=device)
    xd = torch.from_numpy(np.ascontiguousarray(acc)).to(fc.device)
    out = torch.empty((n, h, w, fc.out_wpp), dtype=torch.int64, device=fc.device)
    fc.run(n, h, w, x_f64=xd, bits=out)
    return BitTensor(n, h, w, c, _dev_to_words(out), (ChannelSegment(0, c),))


def xor_popcount_rows(a, b, threads: int = 1, *, device=None) -> np.ndarray:
    """out[m, n] = sum_w popc(a[m, w] ^ b[n, w]) (``kernels.py:114-147``)."""
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[1]:
        raise ValueError(f"row matrices must share word width, got {a.shape} vs {b.shape}")
    dev = cuda_device(device)
    out = torch.empty((a.shape[0], b.shape[0]), dtype=torch.int32, device=dev)
    if out.numel():
        ad, bd = _words_to_dev(a, dev), _words_to_dev(b, dev)
        _lib.call("mbu_xor_popcount_rows", _ptr(ad), _ptr(bd), _ptr(out), a.shape[0], b.shape[0],
                  a.shape[1], _stream(dev))
    return out.cpu().numpy()


def bit_gemm(a: PackedBitMatrix, b_pos: PackedBitMatrix, b_neg, k_true: int, threads: int = 1,
             *, device=None) -> np.ndarray:
    """Exact M x N product of packed rows (``bitcore.py:265-294``), on the GPU."""
    if a.n_lanes != b_pos.n_lanes:
        raise LayoutError(f"K mismatch: A has {a.n_lanes} lanes, B has {b_pos.n_lanes}")
    if a.n_lanes % 128:
        raise LayoutError(f"K = {a.n_lanes} lanes is not 128-block aligned")
    if not 0 <= k_true <= a.n_lanes:
        raise LayoutError(f"k_true = {k_true} outside [0, {a.n_lanes}]")
    if b_neg is not None:
        if b_neg.n_lanes != b_pos.n_lanes or b_neg.n_rows != b_pos.n_rows:
            raise LayoutError("pos/neg weight matrices must share shape")
        if np.any(b_pos.words & b_neg.words):
            raise PlaneOverlapError("a weight lane is set in both pos and neg planes")
        return (xor_popcount_rows(a.words, b_neg.words, device=device)
                - xor_popcount_rows(a.words, b_pos.words, device=device))
    d = xor_popcount_rows(a.words, b_pos.words, device=device)
    return (np.int32(k_true) - 2 * d).astype(np.int32)


def argmax_classes(logits, *, device=None):
    """Class map of a multi-class head (an extra on
    top of the reference's per-channel ``logits >= 0`` mask): uint8
    (n, H, W) = ``numpy.argmax(logits, axis=-1)``, computed by
    ``mbu_argmax``. A CUDA tensor stays on its device; anything else is
    uploaded and the result returned as a NumPy array."""
    on_dev = isinstance(logits, torch.Tensor) and logits.is_cuda
    dev = logits.device if on_dev else cuda_device(device)
    t = logits if on_dev else torch.from_numpy(np.ascontiguousarray(logits, dtype=np.float64)).to(dev)
    if t.dtype != torch.float64 or t.ndim < 1:
        raise ShapeError(f"logits must be float64 with a channel axis, got {t.dtype} {tuple(t.shape)}")
    t = t.contiguous()
    c = t.shape[-1]
    out = torch.empty(t.shape[:-1], dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        _lib.call("mbu_argmax", _ptr(t), out.numel(), c, _ptr(out), _stream(dev))
    return out if on_dev else out.cpu().numpy()


def pack_mask_bits(mask, *, out=None):
    """Bit-pack a device uint8 mask (n, ...) per frame on the GPU (``mbu_pack_mask``):
    the result row f equals ``numpy.packbits(mask[f].ravel(), bitorder="little")``
    (1 bit per pixel: 256 KB per 1024x2048 frame instead of 2 MB)."""
    if not (isinstance(mask, torch.Tensor) and mask.is_cuda and mask.dtype == torch.uint8):
        raise ShapeError("pack_mask_bits takes a uint8 CUDA tensor")
    m = mask.contiguous()
    n = m.shape[0]
    per = m[0].numel() if n else 0
    if out is None:
        out = torch.empty((n, (per + 7) // 8), dtype=torch.uint8, device=m.device)
    elif tuple(out.shape) != (n, (per + 7) // 8) or out.dtype != torch.uint8 or not out.is_contiguous():
        raise ShapeError(f"packed output must be contiguous uint8 {(n, (per + 7) // 8)}")
    with torch.cuda.device(m.device):
        _lib.call("mbu_pack_mask", _ptr(m), n, per, _ptr(out), _stream(m.device))
    return out


def decode_raster(raster, maxval: int, *, out=None, device=None):
    """Netpbm samples -> float64 image on the GPU (``mbu_decode_raster``):
    ``sample / maxval``, bit-identical to ``read_image`` / the reference's
    ``imageio.read_image`` (imageio.py:59-83). ``raster`` is what
    ``imageio.read_raster`` returns (u8 (n, h, w, c), or (n, h, w, c, 2)
    big-endian byte pairs) as a NumPy array or a CUDA uint8 tensor; ``out``
    an optional float64 CUDA tensor of shape (n, h, w, c)."""
    on_dev = isinstance(raster, torch.Tensor) and raster.is_cuda
    dev = raster.device if on_dev else cuda_device(device)
    r = raster if on_dev else torch.from_numpy(np.ascontiguousarray(raster, dtype=np.uint8)).to(dev)
    if r.dtype != torch.uint8:
        raise ShapeError(f"raster must be uint8, got {r.dtype}")
    r = r.contiguous()
    bps = 2 if maxval > 255 else 1
    shape = tuple(r.shape[:-1]) if bps == 2 else tuple(r.shape)
    if bps == 2 and r.shape[-1] != 2:
        raise ShapeError("16-bit rasters carry a trailing axis of 2 bytes")
    if out is None:
        out = torch.empty(shape, dtype=torch.float64, device=dev)
    elif tuple(out.shape) != shape or out.dtype != torch.float64 or not out.is_contiguous():
        raise ShapeError(f"out must be a contiguous float64 tensor of shape {shape}")
    with torch.cuda.device(dev):
        _lib.call("mbu_decode_raster", _ptr(r), out.numel(), bps, int(maxval), _ptr(out), _stream(dev))
    return out


def quantize_weights(w, state: str, ternary_t: float = 0.7, *, device=None) -> np.ndarray:
    """``ternarize_values`` / ``binarize_values`` (quantizer.py:86-110) on the
    GPU (``mbu_quantize_weights``): dense int8 {-1, 0, +1} weights. The
    ternary threshold ``delta = t * mean|w|`` is the host's numpy float64
    reduction, as in the reference, so every element lands identically;
    already-ternary tensors pass through unchanged."""
    from .errors import ValueAlphabetError
    from .graph import MASKED as MASKED_STATE
    from .quantizer import _exactly

    w = np.asarray(w)
    if w.size == 0:
        raise ShapeError(f"cannot {'ternarize' if state == MASKED_STATE else 'binarize'} an empty tensor")
    delta = 0.0
    if state == MASKED_STATE:
        if ternary_t < 0:
            raise ValueAlphabetError(f"threshold factor must be >= 0, got {ternary_t}")
        if _exactly(w, (-1, 0, 1)):
            return w.astype(np.int8)
        delta = float(ternary_t * np.abs(w).mean(dtype=np.float64))
    dev = cuda_device(device)
    with torch.cuda.device(dev):
        # float32 stays float32 on the wire; anything else (float64, float16, ints) is
        # widened exactly to float64 -- the kernel compares in float64 either way, as
        # numpy does against the float64 delta (no narrowing, e.g. -1e-50 keeps its sign)
        f32 = w.dtype == np.float32
        src = torch.from_numpy(np.ascontiguousarray(w, dtype=np.float32 if f32 else np.float64)).to(dev)
        out = torch.empty(src.shape, dtype=torch.int8, device=dev)
        _lib.call("mbu_quantize_weights" if f32 else "mbu_quantize_weights_f64", _ptr(src), src.numel(),
                  0 if state == MASKED_STATE else 1, delta, _ptr(out), _stream(dev))
        return out.cpu().numpy()


def fuse_bn_sign(gamma, beta, mean, var, eps, bias=None, *, device=None) -> FusedThreshold:
    """``fuse_bn_sign`` (layers.py:455-505) on the GPU (``mbu_fuse_bn_sign``):
    one thread per channel bisects the int32 range against the float64
    predicate; same validation and errors as the reference."""
    from .errors import ValueAlphabetError

    gamma, beta, mean, var = (np.asarray(a, dtype=np.float64) for a in (gamma, beta, mean, var))
    c = gamma.shape[0]
    if not (beta.shape == mean.shape == var.shape == (c,)):
        raise ShapeError("batchnorm vectors must share one channel axis")
    b = np.zeros(c) if bias is None else np.asarray(bias, dtype=np.float64)
    if b.shape != (c,):
        raise ShapeError(f"bias shape {b.shape} != ({c},)")
    if np.any(var < 0):
        raise ValueAlphabetError("variance must be nonnegative")
    if not np.isfinite(np.stack([gamma, beta, mean, var, b])).all() or not (eps > 0 and np.isfinite(eps)):
        raise ValueAlphabetError("batchnorm parameters must be finite with eps > 0")
    dev = cuda_device(device)
    with torch.cuda.device(dev):
        ts = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (gamma, beta, mean, var, b)]
        thr = torch.empty(c, dtype=torch.int32, device=dev)
        codes = torch.empty(c, dtype=torch.uint8, device=dev)
        _lib.call("mbu_fuse_bn_sign", *(_ptr(t) for t in ts[:4]), float(eps), _ptr(ts[4]), c,
                  _ptr(thr), _ptr(codes), _stream(dev))
        return FusedThreshold(thr.cpu().numpy(), codes.cpu().numpy())
