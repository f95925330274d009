"""Reference-made parity fixtures at the BENCHMARKED shapes (config 3 and 5).

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src:. NUMBA_CACHE_DIR=/tmp/nb \
        PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_big.py [config3|config5]

Every digest here comes out of ``bitunet.graph.forward``
(``/root/reference/pkg/src/bitunet/graph.py:413-458``, bitunet 0.1.0, numpy
2.3.5, numba 0.65.0) run on full frames:

* ``forward_1024x2048.npz`` — config 3 frames 0 and 7 of bench.py's image
  recipe (``bench_frame``) through the bench model (``live_bundle`` seed 0)
  and through the reference generator (``synthesize_bundle`` seed 0).
* ``forward_2160x3840.npz`` — config 5: one 4K frame (``bench_frame(0, 2160,
  3840)``) through ``live_bundle`` seed 0 at that extent.

Per frame: SHA-256 of every layer's int32 accumulators and packed output
words (``trace``), the mask, the logits' SHA-256 plus a strided logits sample
and per-frame float statistics (the GPU logits are compared against those
within the reference's 1e-9 tolerance, verify.py:23).
"""

from __future__ import annotations

import gc
import hashlib
import sys
import time
from pathlib import Path

import numpy as np

import bitunet as R  # the reference

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2601_11660_b200 import quantizer as Q  # noqa: E402  (live generator only)
from paper_2601_11660_b200.quantizer import bench_frame  # noqa: E402

OUT = Path(__file__).resolve().parent
LOGIT_STRIDE = 997  # every 997th logit is stored verbatim


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def to_ref_bundle(mine):
    rb = R.WeightBundle()
    for name, e in mine.entries.items():
        rb.add(R.BundleEntry(name, e.kind, e.weights, bias=e.bias, gamma=e.gamma, beta=e.beta,
                             mean=e.mean, var=e.var, eps=e.eps))
    return rb


def put(arrays, key, text):
    arrays[key] = np.frombuffer(text.encode(), np.uint8)


def run(arrays, tag, cfg, bundle, frames, h, w, threads):
    model = R.build(cfg, bundle)
    for f in frames:
        img = bench_frame(f, h, w)[None]
        t0 = time.time()
        res = R.forward(model, img, threads=threads, trace=True)
        key = f"{tag}/f{f}"
        for name, rec in res.trace.items():
            if name == "mask":
                continue
            out, acc = rec["out"], rec["acc"]
            if hasattr(out, "words"):
                put(arrays, f"{key}/{name}/out_sha", sha(out.words))
            if acc is not None and np.issubdtype(np.asarray(acc).dtype, np.integer):
                put(arrays, f"{key}/{name}/acc_sha", sha(acc))
        arrays[f"{key}/mask"] = np.packbits(res.mask.reshape(-1))
        put(arrays, f"{key}/logits_sha", sha(res.logits))
        lg = res.logits.reshape(-1)
        arrays[f"{key}/logits_sample"] = lg[::LOGIT_STRIDE].copy()
        arrays[f"{key}/logits_stats"] = np.array([lg.sum(), np.abs(lg).sum(), lg.min(), lg.max()])
        print(key, f"{time.time() - t0:.1f}s", "mask mean", float(res.mask.mean()), flush=True)
        del res, img, lg
        gc.collect()


def config3(threads):
    arrays = {}
    cfg = R.UNetConfig(height=1024, width=2048)
    run(arrays, "live0", cfg, to_ref_bundle(Q.live_bundle(cfg, np.random.default_rng(0))),
        (0, 7), 1024, 2048, threads)
    run(arrays, "synth0", cfg, R.synthesize_bundle(cfg, np.random.default_rng(0)),
        (0, 7), 1024, 2048, threads)
    np.savez_compressed(OUT / "forward_1024x2048.npz", **arrays)


def config5(threads):
    arrays = {}
    cfg = R.UNetConfig(height=2160, width=3840)
    run(arrays, "live0", cfg, to_ref_bundle(Q.live_bundle(cfg, np.random.default_rng(0))),
        (0,), 2160, 3840, threads)
    np.savez_compressed(OUT / "forward_2160x3840.npz", **arrays)


if __name__ == "__main__":
    import os

    which = sys.argv[1:] or ["config3", "config5"]
    thr = os.cpu_count() or 1
    for w in which:
        {"config3": config3, "config5": config5}[w](thr)
