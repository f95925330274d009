"""Run eager MBU-Net forwards at the bench workload, for ncu captures.

    ncu ... python tools/profile_forward.py [--batch 8] [--reps 1]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2601_11660_b200 as mb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--height", type=int, default=1024)
ap.add_argument("--width", type=int, default=2048)
a = ap.parse_args()
cfg = mb.UNetConfig(height=a.height, width=a.width)
model = mb.build(cfg, mb.live_bundle(cfg, np.random.default_rng(0)))
eng = mb.Engine(model, batch=a.batch, use_graph=False)
eng.image.copy_(torch.rand(eng.shape, dtype=torch.float64, device=eng.device))
for _ in range(a.reps):
    eng.run()
torch.cuda.synchronize()
print("done", eng.launches_per_run)
