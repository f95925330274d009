"""Float bundles -> ternary/binary weights + fused thresholds (build time).

Host-side restatement of the parts of ``pkg/src/bitunet/quantizer.py`` that
``build`` and the parity fixtures need: the quantization rules
(``ternarize_values`` ``:86-102``, ``binarize_values`` ``:105-110``), the
bundle containers (``:171-251``), ``quantize_bundle`` (``:254-309``),
``dense_records`` (``:312-321``) and ``synthesize_bundle`` (``:324-370``).

``synthesize_bundle`` draws from the generator in exactly the reference's
order, so a seed reproduces the reference's bundle bit-for-bit; the GPU box
(which has no reference installed) can therefore rebuild the same models the
golden fixtures were made from. :func:`live_bundle` is the
activation-preserving variant of SURVEY.md §8(d).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import BundleError, ShapeError, ValueAlphabetError
from .layers import FusedThreshold, fuse_bn_sign

__all__ = [
    "DEFAULT_EPS",
    "DEFAULT_TERNARY_T",
    "BundleEntry",
    "WeightBundle",
    "PreparedLayer",
    "ternarize_values",
    "binarize_values",
    "quantize_bundle",
    "dense_records",
    "synthesize_bundle",
    "live_bundle",
]

DEFAULT_EPS = 1e-5
DEFAULT_TERNARY_T = 0.7


def _exactly(w, alphabet) -> bool:
    w = np.asarray(w)
    return bool(np.isin(w, alphabet).all()) if w.size else True


def ternarize_values(w, t: float = DEFAULT_TERNARY_T) -> np.ndarray:
    """delta = t*mean|w|; w > delta -> +1, w < -delta -> -1, else 0."""
    w = np.asarray(w)
    if w.size == 0:
        raise ShapeError("cannot ternarize an empty tensor")
    if t < 0:
        raise ValueAlphabetError(f"threshold factor must be >= 0, got {t}")
    if _exactly(w, (-1, 0, 1)):
        return w.astype(np.int8)
    delta = t * np.abs(w).mean(dtype=np.float64)
    return ((w > delta).astype(np.int8) - (w < -delta).astype(np.int8)).astype(np.int8)


def binarize_values(w) -> np.ndarray:
    """sign(w) with sign(0) = +1."""
    w = np.asarray(w)
    if w.size == 0:
        raise ShapeError("cannot binarize an empty tensor")
    return np.where(w >= 0, 1, -1).astype(np.int8)


@dataclass(eq=False)
class BundleEntry:
    name: str
    kind: str
    weights: np.ndarray
    bias: np.ndarray | None = None
    gamma: np.ndarray | None = None
    beta: np.ndarray | None = None
    mean: np.ndarray | None = None
    var: np.ndarray | None = None
    eps: float | None = None

    @property
    def has_bn(self) -> bool:
        return self.gamma is not None

    def bn_tuple(self) -> tuple:
        f = lambda v: np.asarray(v, dtype=np.float64)  # noqa: E731
        eps = DEFAULT_EPS if self.eps is None else float(self.eps)
        return (f(self.gamma), f(self.beta), f(self.mean), f(self.var), eps)


@dataclass(eq=False)
class WeightBundle:
    entries: dict = field(default_factory=dict)

    def __contains__(self, name) -> bool:
        return name in self.entries

    def __getitem__(self, name) -> BundleEntry:
        return self.entries[name]

    def add(self, entry: BundleEntry) -> None:
        self.entries[entry.name] = entry


@dataclass(eq=False)
class PreparedLayer:
    name: str
    kind: str
    weights: np.ndarray
    bias: np.ndarray | None = None
    bn: tuple | None = None
    threshold: FusedThreshold | None = None


def quantize_bundle(bundle, config, ternary_t: float = DEFAULT_TERNARY_T, *, device=None) -> dict:
    """Quantize every conv of ``bundle`` per the config's PrecisionMap.

    ``device`` (an extra): run the element-wise
    ternarize / binarize and the per-channel ``fuse_bn_sign`` searches on that
    CUDA device (``ops.quantize_weights`` / ``ops.fuse_bn_sign``); the result
    is identical to the host path."""
    if device is not None:
        from . import ops

        quant = lambda w, state: ops.quantize_weights(w, state, ternary_t, device=device)  # noqa: E731
        fuse = lambda *bn, bias: ops.fuse_bn_sign(*bn, bias=bias, device=device)  # noqa: E731
    else:
        quant = lambda w, state: ternarize_values(w, ternary_t) if state == "masked" else binarize_values(w)  # noqa: E731
        fuse = lambda *bn, bias: fuse_bn_sign(*bn, bias=bias)  # noqa: E731
    from .graph import MASKED, layer_specs

    out = {}
    for e in layer_specs(config):
        if e.kind not in ("float-conv", "bit-conv", "bit-tconv"):
            continue
        if e.name not in bundle:
            raise BundleError(f"bundle is missing layer {e.name!r}")
        be = bundle[e.name]
        want_kind = "tconv" if e.kind == "bit-tconv" else "conv"
        if be.kind != want_kind:
            raise BundleError(f"layer {e.name!r} has kind {be.kind!r}, expected {want_kind!r}")
        s = e.conv
        want = (s.c_out, s.kernel_h, s.kernel_w, s.c_in)
        w = np.asarray(be.weights)
        if w.shape != want:
            raise ShapeError(f"layer {e.name!r} weights shape {w.shape}, expected {want}")
        if e.has_bn != be.has_bn:
            raise BundleError(
                f"layer {e.name!r} {'must' if e.has_bn else 'must not'} carry batchnorm"
            )
        bias = None if be.bias is None else np.asarray(be.bias, dtype=np.float64)
        if bias is not None and bias.shape != (s.c_out,):
            raise ShapeError(f"layer {e.name!r} bias shape {bias.shape}, expected ({s.c_out},)")
        if e.kind == "float-conv":
            out[e.name] = PreparedLayer(e.name, "float", w.astype(np.float64), bias,
                                        be.bn_tuple() if be.has_bn else None)
            continue
        state = MASKED if e.label == "stem2" else config.precision.state(e.label)
        dense = quant(w, state)
        bn = be.bn_tuple()
        out[e.name] = PreparedLayer(e.name, state, dense, bias, bn, fuse(*bn, bias=bias))
    return out


def dense_records(prepared: dict, config) -> dict:
    """PreparedLayers -> the dense record dicts the oracle consumes."""
    recs = {}
    for name, p in prepared.items():
        r = {"w": p.weights, "bias": p.bias, "bn": p.bn}
        if p.threshold is not None:
            r["threshold"] = (p.threshold.thresholds, p.threshold.codes)
            r["pad_value"] = config.pad_value
        recs[name] = r
    return recs


def synthesize_bundle(config, rng: np.random.Generator, negative_gamma_rate: float = 0.15,
                      zero_gamma_rate: float = 0.0) -> WeightBundle:
    """Random bundle with the reference's draw order (``quantizer.py:324-370``)."""
    from .graph import layer_specs

    bundle = WeightBundle()
    for e in layer_specs(config):
        if e.kind not in ("float-conv", "bit-conv", "bit-tconv"):
            continue
        s = e.conv
        k = s.kernel_h * s.kernel_w * s.c_in
        weights = rng.standard_normal((s.c_out, s.kernel_h, s.kernel_w, s.c_in)).astype(np.float32)
        bias = rng.standard_normal(s.c_out).astype(np.float32) if e.has_bias else None
        bn = {}
        if e.has_bn:
            gamma = rng.uniform(0.3, 1.5, s.c_out)
            gamma[rng.random(s.c_out) < negative_gamma_rate] *= -1.0
            gamma[rng.random(s.c_out) < zero_gamma_rate] = 0.0
            bn["gamma"] = gamma.astype(np.float32)
            bn["beta"] = rng.standard_normal(s.c_out).astype(np.float32)
            bn["mean"] = (rng.uniform(-0.5, 0.5, s.c_out) * k).astype(np.float32)
            bn["var"] = rng.uniform(0.5, max(1.0, (k / 3) ** 2), s.c_out).astype(np.float32)
            bn["eps"] = DEFAULT_EPS
        kind = "tconv" if e.kind == "bit-tconv" else "conv"
        bundle.add(BundleEntry(e.name, kind, weights, bias=bias, **bn))
    return bundle


def live_bundle(config, rng: np.random.Generator) -> WeightBundle:
    """Activation-preserving bundle ("live generator").

    The reference generator centres BN far outside the accumulator's actual
    +-O(sqrt K) spread, so almost every channel is constant and mask parity
    is nearly vacuous. This variant redraws the BN statistics at the
    accumulator's real scale: for bit layers with K_eff = 0.58*K,
    mean ~ N(0, 0.5*sqrt(K_eff)), var ~ U(0.5, 2)*K_eff, beta ~ N(0, 0.3);
    for the stem mean ~ N(0, 1), var ~ U(0.5, 2); the head bias is 0.
    """
    from .graph import layer_specs

    bundle = synthesize_bundle(config, rng)
    for e in layer_specs(config):
        if e.kind not in ("float-conv", "bit-conv", "bit-tconv") or e.name not in bundle:
            continue
        be = bundle[e.name]
        c = e.conv.c_out
        if e.name == "head":
            be.bias = np.zeros(c, dtype=np.float32)
            continue
        if not be.has_bn:
            continue
        if e.kind == "float-conv":
            be.mean = rng.normal(0.0, 1.0, c).astype(np.float32)
            be.var = rng.uniform(0.5, 2.0, c).astype(np.float32)
        else:
            k_eff = 0.58 * e.conv.kernel_h * e.conv.kernel_w * e.conv.c_in
            be.mean = rng.normal(0.0, 0.5 * np.sqrt(k_eff), c).astype(np.float32)
            be.var = (rng.uniform(0.5, 2.0, c) * k_eff).astype(np.float32)
            be.beta = rng.normal(0.0, 0.3, c).astype(np.float32)
    return bundle


def bench_frame(index: int, height: int, width: int) -> np.ndarray:
    """Synthetic frame ``index`` of the benchmark stream: float64 (H, W, 3) in [0, 1).

    ``bench.py`` fills its batches with these and the big-shape golden
    fixtures (``tests/golden/make_golden_big.py``) are the reference's forward
    of the same frames, so the benchmarked inputs are parity-pinned.
    """
    return np.random.default_rng(1000 + index).random((height, width, 3))
