"""Bind this engine into an imported ``bitunet`` at the reference's own plug point.

``bitunet.graph.forward`` (``pkg/src/bitunet/graph.py:413-458``) dispatches
every layer through module-level names (``conv_forward``, ``apply_threshold``,
``maxpool2``, ``float_conv`` ...), and the package re-exports those names
(``pkg/src/bitunet/__init__.py:47-69``), so rebinding them is how a
``bitunet`` user swaps the compute path without touching call sites.
:func:`install` does that rebinding for every ``bitunet.*`` module that bound
one of the originals, with thin adapters that hand the GPU results back as
the reference's own types (``bitunet.bitcore.BitTensor``,
``bitunet.graph.ForwardResult``), so ``isinstance`` checks in the reference
(graph.py:435, verify.py:43) keep working.

Two levels, both on by default:

* ``layers=True`` — the layer functions (``conv_forward``,
  ``transposed_conv_forward``, ``apply_threshold``, ``maxpool2``,
  ``float_conv``, ``float_bn_sign``, ``xor_popcount_rows``, ``bit_gemm``):
  the reference's interpreter loop runs, every layer on the GPU;
* ``forward=True`` — ``graph.forward`` itself: the whole network as one
  native plan on the GPU (``runtime.forward``).

The reference's dense oracle (``bitunet.oracle``) is never rebound, so the
reference's own verification (``verify.verify_model``) keeps checking the
GPU results against it. :func:`install` returns a callable that restores the
original bindings. This is what ``tests/test_gpu_conformance.py`` runs the
reference's test suite through, and what INTEGRATION.md §2 describes.
"""

from __future__ import annotations

import sys

__all__ = ["install", "to_reference"]

_NEVER = ("bitunet.oracle",)  # the checker stays the reference's own


def to_reference(obj, R=None):
    """Our BitTensor / trace dict / ForwardResult as the reference's types."""
    from .bitcore import BitTensor

    if R is None:
        import bitunet as R  # noqa: N812
    if isinstance(obj, BitTensor):
        segs = tuple(R.bitcore.ChannelSegment(s.lane_offset, s.count) for s in obj.segments)
        return R.bitcore.BitTensor(obj.n, obj.h, obj.w, obj.c, obj.words, segs)
    if isinstance(obj, dict):
        return {k: to_reference(v, R) for k, v in obj.items()}
    return obj


def _adapters(R):
    from . import ops, runtime

    def conv_forward(x, weights, spec, threads=1):
        return ops.conv_forward(x, weights, spec, threads)

    def transposed_conv_forward(x, weights, spec, threads=1):
        return ops.transposed_conv_forward(x, weights, spec, threads)

    def apply_threshold(acc, t):
        return to_reference(ops.apply_threshold(acc, t), R)

    def maxpool2(x):
        return to_reference(ops.maxpool2(x), R)

    def float_conv(x, w, bias, spec):
        return ops.float_conv(x, w, bias, spec)

    def float_bn_sign(acc, gamma, beta, mean, var, eps, bias=None):
        return to_reference(ops.float_bn_sign(acc, gamma, beta, mean, var, eps, bias), R)

    def xor_popcount_rows(a, b, threads=1):
        return ops.xor_popcount_rows(a, b, threads)

    def bit_gemm(a, b_pos, b_neg, k_true, threads=1):
        return ops.bit_gemm(a, b_pos, b_neg, k_true, threads)

    def forward(model, image, threads=1, trace=False):
        res = runtime.forward(model, image, threads, trace)
        return R.graph.ForwardResult(res.logits, res.mask, to_reference(res.trace, R))

    layer_fns = {
        R.layers.conv_forward: conv_forward,
        R.layers.transposed_conv_forward: transposed_conv_forward,
        R.layers.apply_threshold: apply_threshold,
        R.layers.maxpool2: maxpool2,
        R.layers.float_conv: float_conv,
        R.layers.float_bn_sign: float_bn_sign,
        R.kernels.xor_popcount_rows: xor_popcount_rows,
        R.bitcore.bit_gemm: bit_gemm,
    }
    return layer_fns, {R.graph.forward: forward}


def install(R=None, *, layers: bool = True, forward: bool = True):
    """Rebind ``bitunet``'s compute functions to the GPU engine; returns ``restore()``."""
    if R is None:
        import bitunet as R  # noqa: N812
    layer_fns, fwd = _adapters(R)
    repl = {}
    if layers:
        repl.update(layer_fns)
    if forward:
        repl.update(fwd)
    by_id = {id(k): v for k, v in repl.items()}
    undo = []
    for name, mod in list(sys.modules.items()):
        if mod is None or not (name == "bitunet" or name.startswith("bitunet.")):
            continue
        if name.startswith(_NEVER):
            continue
        for attr, val in list(vars(mod).items()):
            new = by_id.get(id(val))
            if new is not None:
                setattr(mod, attr, new)
                undo.append((mod, attr, val))

    def restore():
        for mod, attr, val in reversed(undo):
            setattr(mod, attr, val)

    restore.rebound = [(m.__name__, a) for m, a, _ in undo]
    return restore
