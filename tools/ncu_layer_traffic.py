"""Per-layer DRAM traffic and duration of one eager forward, from
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv
over tools/profile_forward.py (--reps 1: Engine init runs one forward, then one more is
profiled; the second forward's launches are matched to the layers in order).
usage: python tools/ncu_layer_traffic.py gpurun_out/traffic.csv > profiles/rX_layer_traffic.md
Algorithmic bytes per layer (8 x 1024 x 2048 batch): packed input read once + packed output
written once (+ the f64 image for the stem, f64 logits + u8 mask for the head)."""
import csv
import io
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

txt = open(sys.argv[1]).read()
rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
per = defaultdict(dict)
names = {}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}
for r in rows:
    per[int(r["ID"])][r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
    names[int(r["ID"])] = r["Kernel Name"]
ids = sorted(per)
import numpy as np  # noqa: E402

import paper_2601_11660_b200 as mb  # noqa: E402

cfg = mb.UNetConfig(height=1024, width=2048)
model = mb.build(cfg, mb.synthesize_bundle(cfg, np.random.default_rng(0)))
layers = [l for l in model.layers if l.kind != "concat"]
ids = ids[-len(layers):]  # the profiled (second) forward
N, H, W = 8, 1024, 2048
h, w, wpp_in = H, W, None
print("| layer | kernel | ms | DRAM read MB | DRAM write MB | algorithmic MB | DRAM / algorithmic | GB/s |")
print("|---|---|---|---|---|---|---|---|")
wpp = {}
for l, i in zip(layers, ids):
    m = per[i]
    rd, wr, t = m["dram__bytes_read.sum"], m["dram__bytes_write.sum"], m["gpu__time_duration.sum"]
    s = l.spec
    if l.kind == "float-conv" and l.name == "stem":
        alg = N * H * W * 3 * 8 + N * H * W * 16
        h, w = H, W
    elif l.kind == "maxpool":
        alg = N * h * w * 16 * (wpp_last // 2) + N * (h // 2) * (w // 2) * 16 * (wpp_last // 2)
        h, w = h // 2, w // 2
    elif l.kind == "float-conv":
        alg = N * h * w * 16 + N * h * w * (8 + 1)
    else:
        cin_w = ((s.c_in + 127) // 128) * 16
        if l.kind.endswith("tconv"):
            ho, wo = h * 2, w * 2
        else:
            ho, wo = h, w
        alg = N * h * w * cin_w + N * ho * wo * ((s.c_out + 127) // 128) * 16
        h, w = ho, wo
    if l.kind != "maxpool" and l.kind != "float-conv":
        wpp_last = ((s.c_out + 127) // 128) * 2
    elif l.name == "stem":
        wpp_last = 2
    kn = names[i].split("(")[0].replace("void ", "")[:40]
    print(f"| {l.name} | `{kn}` | {t * 1e3:.3f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | {alg / 1e6:.1f} | "
          f"{(rd + wr) / alg:.2f} | {(rd + wr) / t / 1e9:.0f} |")
