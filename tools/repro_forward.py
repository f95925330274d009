"""Forward of the default network at a given shape (debug / compute-sanitizer repro)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2601_11660_b200 as mb  # noqa: E402

h, w, n = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (256, 512, 1)
cfg = mb.UNetConfig(height=h, width=w)
model = mb.build(cfg, mb.live_bundle(cfg, np.random.default_rng(0)))
img = np.random.default_rng(1).random((n, h, w, 3))
res = mb.forward(model, img)
torch.cuda.synchronize()
print("ok", res.mask.mean())
