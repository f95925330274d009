"""Run every bit conv layer of the default network alone (random packed input of
its bench shape) in a fresh process each; reports which launch fails or hangs.
usage: python tools/layer_sweep.py [H W N]"""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
H, W, N = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (1024, 2048, 1)
CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2601_11660_b200 as mb
from paper_2601_11660_b200.ops import ConvHandle
from paper_2601_11660_b200.bitcore import segment_lanes
H, W, N, idx = %d, %d, %d, %d
cfg = mb.UNetConfig(height=H, width=W)
model = mb.build(cfg, mb.live_bundle(cfg, np.random.default_rng(0)))
dm = mb.runtime.DeviceModel(model, torch.device('cuda', 0))
dm.plan(N, H, W, False)
layer = model.layers[idx]
info = dm.layer_info(idx - 1) if model.layers[idx - 1].kind != 'concat' else None
segs = dm.out_segments[idx - 1]
h, w = dm.layer_info(idx - 1)['h'], dm.layer_info(idx - 1)['w']
cv = ConvHandle(layer.weights, layer.spec, segs, layer.threshold, transposed=layer.kind.endswith('tconv'))
wpp = segment_lanes(segs) // 64
x = torch.randint(-2**62, 2**62, (N, h, w, wpp), dtype=torch.int64, device='cuda')
ho, wo = cv.out_extent(h, w)
out = torch.empty((N, ho, wo, cv.out_wpp), dtype=torch.int64, device='cuda')
cv.run(x, N, h, w, bits=out)
torch.cuda.synchronize()
print('ok')
"""
sys.path.insert(0, str(ROOT))
import paper_2601_11660_b200 as mb  # noqa: E402  (names only)
import numpy as np  # noqa: E402
cfg = mb.UNetConfig(height=H, width=W)
model = mb.build(cfg, mb.synthesize_bundle(cfg, np.random.default_rng(0)))
for i, l in enumerate(model.layers):
    if l.kind not in ("masked-conv", "binary-conv", "masked-tconv", "binary-tconv") or i == 0:
        continue
    try:
        r = subprocess.run([sys.executable, "-c", CHILD % (str(ROOT), H, W, N, i)], capture_output=True,
                           text=True, timeout=60)
        res = "ok" if r.returncode == 0 else (r.stderr.strip().splitlines() or ["?"])[-1][:120]
    except subprocess.TimeoutExpired:
        res = "HANG"
    print(json.dumps({"layer": l.name, "kind": l.kind, "result": res}), flush=True)
