"""Per-tile MMA / epilogue / producer timestamps of CTA 0 for every conv_tc launch of one
forward (stderr). Needs a library built with -DMBU_TIMELINE, e.g.
  nvcc ... -DMBU_TIMELINE -c csrc/conv_tc.cu; link with the other objects into build/ab/tl.so
  MBU_LIB=build/ab/tl.so python tools/timeline_probe.py 2> timeline.txt
"""
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
