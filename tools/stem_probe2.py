"""Stem kernel alone through FloatConvHandle: CUDA-event timing per launch."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2601_11660_b200 as mb  # noqa: E402
from paper_2601_11660_b200 import _lib  # noqa: E402
from paper_2601_11660_b200.ops import FloatConvHandle  # noqa: E402

cfg = mb.UNetConfig(height=1024, width=2048)
model = mb.build(cfg, mb.live_bundle(cfg, np.random.default_rng(0)))
L = model.layers[0]
fc = FloatConvHandle(L.weights, L.bias, L.spec, bn=L.bn)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
x = torch.rand((n, 1024, 2048, 3), dtype=torch.float64, device="cuda")
out = torch.zeros((n, 1024, 2048, 2), dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for mode in (0, 1):
    _lib.call("mbu_set_option", 2, mode)
    for fl in (0, 1):
        ts = []
        for _ in range(5):
            if fl:
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fc.run(n, 1024, 2048, x_f64=x, bits=out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print("ffma" if mode else "tc", "flush" if fl else "", ["%.4f" % t for t in ts], flush=True)
_lib.call("mbu_set_option", 2, 0)
