"""cProfile of the drop-in forward() at the bench workload (where the host time goes)."""
import cProfile
import pstats
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2601_11660_b200 as mb  # noqa: E402
from paper_2601_11660_b200.quantizer import bench_frame  # noqa: E402

cfg = mb.UNetConfig(height=1024, width=2048)
model = mb.build(cfg, mb.live_bundle(cfg, np.random.default_rng(0)))
imgs = np.stack([bench_frame(i, 1024, 2048) for i in range(8)])
for _ in range(2):
    r = mb.forward(model, imgs, device="cuda:0")
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    r = mb.forward(model, imgs, device="cuda:0")
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
