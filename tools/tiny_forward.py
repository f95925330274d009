"""A tiny MBU-Net forward on cuda:0 checked against the dense oracle (compute-sanitizer target).
usage: python tools/tiny_forward.py [extent] [batch]"""
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2601_11660_b200 as mb  # noqa: E402
from oracle import dense  # noqa: E402

extent = int(sys.argv[1]) if len(sys.argv) > 1 else 32
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = replace(mb.scale_config(mb.UNetConfig(), 4), height=extent, width=extent)
rng = np.random.default_rng(5)
bundle = mb.live_bundle(cfg, rng)
model = mb.build(cfg, bundle)
image = rng.random((n, extent, extent, 3))
res = mb.forward(model, image, trace=True)
eng = mb.Engine(model, batch=n)
import torch  # noqa: E402

eng.image.copy_(torch.from_numpy(image))
eng.run()
torch.cuda.synchronize()
ref = dense.ref_forward(cfg, mb.dense_records(mb.quantize_bundle(bundle, cfg), cfg), image)
assert np.array_equal(res.mask, ref["mask"]) and np.array_equal(eng.mask.cpu().numpy(), ref["mask"])
print("tiny forward ok", res.mask.mean())
