"""Per-tile MMA / epilogue timestamps of CTA 0 (needs a -DMBU_TIMELINE build via MBU_LIB)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2601_11660_b200 as mb  # noqa: E402

cfg = mb.UNetConfig(height=1024, width=2048)
model = mb.build(cfg, mb.live_bundle(cfg, np.random.default_rng(0)))
eng = mb.Engine(model, batch=8, use_graph=False)
eng.image.copy_(torch.rand(eng.shape, dtype=torch.float64, device=eng.device))
with torch.cuda.stream(eng.stream):
    eng._enqueue()
torch.cuda.synchronize()
