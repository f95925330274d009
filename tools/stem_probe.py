"""Time the stem layer alone (eager, CUDA events) in its execution modes."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2601_11660_b200 as mb  # noqa: E402
from paper_2601_11660_b200 import _lib  # noqa: E402

cfg = mb.UNetConfig(height=1024, width=2048)
model = mb.build(cfg, mb.live_bundle(cfg, np.random.default_rng(0)))
eng = mb.Engine(model, batch=8, use_graph=False)
eng.image.copy_(torch.rand(eng.shape, dtype=torch.float64, device=eng.device))
dm = eng.dm
for mode in (0, 1, 0, 1):
    _lib.call("mbu_set_option", 2, mode)
    dm.set_timing(True)
    ts = []
    for _ in range(5):
        with torch.cuda.stream(eng.stream):
            eng._enqueue()
        ts.append(dm.layer_times()[0])
    dm.set_timing(False)
    print("ffma" if mode else "tc", ["%.4f" % t for t in ts], flush=True)
_lib.call("mbu_set_option", 2, 0)
# whole forward, eager, back to back
for k in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(eng.stream)
    for _ in range(10):
        with torch.cuda.stream(eng.stream):
            eng._enqueue()
    e1.record(eng.stream)
    torch.cuda.synchronize()
    print("eager forward ms", e0.elapsed_time(e1) / 10)
