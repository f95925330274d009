"""Generate golden parity fixtures by running the REFERENCE itself.

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src:. NUMBA_CACHE_DIR=/tmp/nb \
        PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Everything written here comes out of ``bitunet`` 0.1.0
(``/root/reference/pkg/src/bitunet``; numpy 2.3.5, numba 0.65.0). The GPU
box has no reference, so these files are what pins both the CPU oracle and
the CUDA path there. Fixtures:

* ``bn_fusion.npz`` — ``fuse_bn_sign`` on 2000 random BN draws, including
  decision points outside int32 and gamma == 0 (criterion 5 style).
* ``layers.npz`` — layer-level cases: dense inputs and weights, the packed
  words the reference builds from them, and ``conv_forward`` /
  ``transposed_conv_forward`` / ``maxpool2`` / ``apply_threshold`` results.
* ``forward_tiny.npz`` — full traces (every layer's acc and packed out words)
  of base-16 models at 16x16 / 32x32 for five precision/pad variants, from
  ``synthesize_bundle(cfg, default_rng(seed))``.
* ``forward_256.npz`` — 1x256x256 default-width models (config 1): logits,
  mask and per-layer SHA-256 digests of acc and out words, for the
  reference generator and for the activation-preserving ("live") bundle.
* ``build_digest.json`` — SHA-256 of every plane / threshold the reference
  ``build`` emits for those models (pins our host-side ``build``).
"""

from __future__ import annotations

import hashlib
import json
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np

import bitunet as R  # the reference
from bitunet import layers as RL
from bitunet.graph import scale_config

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2601_11660_b200 import quantizer as Q  # noqa: E402  (live generator only)

OUT = Path(__file__).resolve().parent


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def bn_fixture():
    rng = np.random.default_rng(20261017)
    c = 2000
    g = rng.normal(size=c) * 10.0 ** rng.integers(-4, 4, c)
    g[rng.random(c) < 0.05] = 0.0
    b = rng.normal(size=c) * 10.0 ** rng.integers(-2, 6, c)
    m = rng.normal(size=c) * 10.0 ** rng.integers(-1, 11, c)
    v = rng.uniform(0, 3, c) * 10.0 ** rng.integers(-6, 8, c)
    bias = rng.normal(size=c) * 10.0 ** rng.integers(-2, 4, c)
    ft = RL.fuse_bn_sign(g, b, m, v, 1e-5, bias)
    np.savez_compressed(OUT / "bn_fusion.npz", gamma=g, beta=b, mean=m, var=v, bias=bias,
                        eps=1e-5, thresholds=ft.thresholds, codes=ft.codes)


def layer_fixture():
    rng = np.random.default_rng(0xBADC0DE)
    arrays = {}
    cases = []
    geoms = [(1, 1, 0), (2, 2, 0), (3, 1, 1), (3, 2, 1)]
    chans = [1, 5, 33, 64, 70, 128, 192, 200, 256]
    i = 0
    for c_in in chans:
        for gi, (k, s, p) in enumerate(geoms):
            for masked in (True, False):
                c_out = int(rng.integers(1, 40)) if (i % 3) else int(rng.choice([32, 64, 96]))
                pad_mode = "zero" if masked and i % 4 == 0 else "neg_one"
                h = w = int(rng.choice([4, 5, 7])) if s == 1 else 6
                x = rng.choice((-1, 1), size=(2, h, w, c_in)).astype(np.int8)
                alph = (-1, 0, 1) if masked else (-1, 1)
                wt = rng.choice(alph, size=(c_out, k, k, c_in)).astype(np.int8)
                xt = R.pack_tensor(x)
                planes = RL.pack_conv_weights(wt, xt.segments, masked=masked)
                spec = RL.ConvSpec(k, k, s, p, c_in, c_out, pad_mode=pad_mode)
                acc = RL.conv_forward(xt, planes, spec)
                key = f"conv{i}"
                arrays[f"{key}_x"] = x
                arrays[f"{key}_w"] = wt
                arrays[f"{key}_acc"] = acc
                arrays[f"{key}_pos"] = (planes.pos if masked else planes).words
                if masked:
                    arrays[f"{key}_neg"] = planes.neg.words
                cases.append(dict(key=key, op="conv", k=k, s=s, p=p, c_in=c_in, c_out=c_out,
                                  masked=masked, pad_mode=pad_mode))
                i += 1
    # non-contiguous segment layout (the concat gap case, test_layers.py:233-242)
    a = rng.choice((-1, 1), size=(1, 5, 6, 6)).astype(np.int8)
    b = rng.choice((-1, 1), size=(1, 5, 6, 130)).astype(np.int8)
    cat = RL.concat_channels(R.pack_tensor(a), R.pack_tensor(b))
    for masked in (True, False):
        wt = rng.choice((-1, 0, 1) if masked else (-1, 1), size=(9, 3, 3, 136)).astype(np.int8)
        planes = RL.pack_conv_weights(wt, cat.segments, masked=masked)
        acc = RL.conv_forward(cat, planes, RL.ConvSpec(3, 3, 1, 1, 136, 9))
        key = f"gap{int(masked)}"
        arrays[f"{key}_words"] = cat.words
        arrays[f"{key}_xa"] = a
        arrays[f"{key}_xb"] = b
        arrays[f"{key}_w"] = wt
        arrays[f"{key}_acc"] = acc
        cases.append(dict(key=key, op="gapconv", masked=masked,
                          segments=[[s.lane_offset, s.count] for s in cat.segments]))
    # transposed convs, k = s in {2, 3}
    for j in range(24):
        k = 2 + j % 2
        c_in = [8, 64, 130, 256][j % 4]
        c_out = [48, 7, 96, 12, 384, 5][j % 6]
        masked = bool(j % 2)
        x = rng.choice((-1, 1), size=(2, 3, 4, c_in)).astype(np.int8)
        wt = rng.choice((-1, 0, 1) if masked else (-1, 1), size=(c_out, k, k, c_in)).astype(np.int8)
        xt = R.pack_tensor(x)
        planes = RL.pack_conv_weights(wt, xt.segments, masked=masked)
        acc = RL.transposed_conv_forward(xt, planes, RL.ConvSpec(k, k, k, 0, c_in, c_out))
        key = f"tconv{j}"
        arrays[f"{key}_x"] = x
        arrays[f"{key}_w"] = wt
        arrays[f"{key}_acc"] = acc
        cases.append(dict(key=key, op="tconv", k=k, c_in=c_in, c_out=c_out, masked=masked))
    # pools
    for j in range(12):
        c = int(rng.integers(1, 300))
        h, w = 2 * int(rng.integers(1, 5)), 2 * int(rng.integers(1, 5))
        x = rng.choice((-1, 1), size=(2, h, w, c)).astype(np.int8)
        key = f"pool{j}"
        arrays[f"{key}_x"] = x
        arrays[f"{key}_out"] = R.maxpool2(R.pack_tensor(x)).words
        cases.append(dict(key=key, op="pool"))
    # thresholds
    codes = np.array([RL.DIR_GE, RL.DIR_LE, RL.CONST_NEG, RL.CONST_POS], dtype=np.uint8)
    for j in range(12):
        c = int(rng.integers(1, 513))
        acc = rng.integers(-10_000, 10_001, size=(1, 2, 3, c)).astype(np.int32)
        t = rng.integers(-10_000, 10_001, size=c).astype(np.int32)
        cc = rng.choice(codes, size=c)
        key = f"thr{j}"
        arrays[f"{key}_acc"] = acc
        arrays[f"{key}_t"] = t
        arrays[f"{key}_codes"] = cc
        arrays[f"{key}_out"] = RL.apply_threshold(acc, RL.FusedThreshold(t, cc)).words
        cases.append(dict(key=key, op="threshold"))
    arrays["cases_json"] = np.frombuffer(json.dumps(cases).encode(), dtype=np.uint8)
    np.savez_compressed(OUT / "layers.npz", **arrays)


TINY_VARIANTS = {
    "all-masked": {},
    "all-binary": {"precision": "binary"},
    "tconvs-masked": {"precision": 0x0F0},
    "stem2-float": {"stem2_float": True},
    "zero-pad": {"pad_mode": "zero"},
}


def tiny_cfg(extent, overrides):
    ov = dict(overrides)
    if ov.get("precision") == "binary":
        ov["precision"] = R.PrecisionMap.all_binary()
    elif "precision" in ov:
        ov["precision"] = R.PrecisionMap.from_config_id(ov["precision"])
    cfg = replace(scale_config(R.UNetConfig(), 4), height=extent, width=extent)
    return replace(cfg, **ov)


def to_ref_bundle(mine):
    rb = R.WeightBundle()
    for name, e in mine.entries.items():
        rb.add(R.BundleEntry(name, e.kind, e.weights, bias=e.bias, gamma=e.gamma, beta=e.beta,
                             mean=e.mean, var=e.var, eps=e.eps))
    return rb


def model_digest(model):
    d = {}
    for l in model.layers:
        if l.threshold is not None:
            d[l.name + ".T"] = sha(l.threshold.thresholds)
            d[l.name + ".codes"] = sha(l.threshold.codes)
        w = l.weights
        if w is None:
            continue
        if hasattr(w, "neg"):
            d[l.name + ".pos"] = sha(w.pos.words)
            d[l.name + ".neg"] = sha(w.neg.words)
        elif hasattr(w, "words"):
            d[l.name + ".plane"] = sha(w.words)
        else:
            d[l.name + ".w"] = sha(np.asarray(w, dtype=np.float64))
    return d


def trace_arrays(prefix, trace, arrays, full=True):
    for name, rec in trace.items():
        if name == "mask":
            arrays[f"{prefix}/mask"] = rec
            continue
        out, acc = rec["out"], rec["acc"]
        if hasattr(out, "words"):
            if full:
                arrays[f"{prefix}/{name}/out"] = out.words
            else:
                arrays[f"{prefix}/{name}/out_sha"] = np.frombuffer(sha(out.words).encode(), np.uint8)
        elif full:
            arrays[f"{prefix}/{name}/out"] = out
        if acc is not None:
            if full:
                arrays[f"{prefix}/{name}/acc"] = acc
            elif np.issubdtype(np.asarray(acc).dtype, np.integer):
                arrays[f"{prefix}/{name}/acc_sha"] = np.frombuffer(sha(acc).encode(), np.uint8)


def forward_fixtures():
    digests = {}
    arrays = {}
    for extent, seed in ((16, 7), (32, 8)):
        for vname, ov in TINY_VARIANTS.items():
            cfg = tiny_cfg(extent, ov)
            bundle = R.synthesize_bundle(cfg, np.random.default_rng(seed))
            model = R.build(cfg, bundle)
            img = np.random.default_rng(seed + 100).random((2, extent, extent, 3))
            res = R.forward(model, img, trace=True)
            key = f"{vname}@{extent}"
            arrays[f"{key}/image"] = img
            arrays[f"{key}/logits"] = res.logits
            trace_arrays(key, res.trace, arrays, full=True)
            digests[key] = model_digest(model)
    np.savez_compressed(OUT / "forward_tiny.npz", **arrays)

    arrays = {}
    cfg = R.UNetConfig(height=256, width=256)
    for gen, seed in (("synth", 1), ("live", 1), ("live", 2)):
        if gen == "synth":
            bundle = R.synthesize_bundle(cfg, np.random.default_rng(seed))
        else:
            bundle = to_ref_bundle(Q.live_bundle(cfg, np.random.default_rng(seed)))
        model = R.build(cfg, bundle)
        img = np.random.default_rng(seed + 1000).random((1, 256, 256, 3))
        res = R.forward(model, img, trace=True)
        key = f"{gen}{seed}@256"
        arrays[f"{key}/logits"] = res.logits
        trace_arrays(key, res.trace, arrays, full=False)
        digests[key] = model_digest(model)
        print(key, "mask mean", res.mask.mean())
    np.savez_compressed(OUT / "forward_256.npz", **arrays)
    (OUT / "build_digest.json").write_text(json.dumps(digests, indent=1, sort_keys=True))


if __name__ == "__main__":
    bn_fixture()
    layer_fixture()
    forward_fixtures()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
