"""Where do the tensor-core stem bits differ from the float64 kernel?"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import paper_2601_11660_b200 as mb  # noqa: E402
from oracle import dense  # noqa: E402
from paper_2601_11660_b200.ops import FloatConvHandle  # noqa: E402
from test_gpu_layers import _stem_bits  # noqa: E402

cuda = torch.device("cuda:0")
rng = np.random.default_rng(5)
x = rng.random((2, 40, 136, 3))
inf_on = len(sys.argv) > 1
if inf_on:
    x[0, 3, 4] = [np.inf, 0.5, 0.5]
w = rng.normal(size=(64, 3, 3, 3))
b = rng.normal(size=64)
g = rng.uniform(-1.5, 1.5, 64)
g[0] = 0.0
be = rng.normal(size=64)
v = rng.uniform(0.5, 2.0, 64)
eps = 1e-5
acc = dense.ref_float_conv(x[1:2], w, b, 1, 1)
sigma = np.sqrt(v + eps)
mean = acc[0, 17, 9, :] + be * sigma / np.where(g == 0, 1.0, g)
fc = FloatConvHandle(w, b, mb.ConvSpec(3, 3, 1, 1, 3, 64), bn=(g, be, mean, v, eps))
tc = _stem_bits(fc, x, cuda, "tc")
gen = _stem_bits(fc, x, cuda, "generic")
A = mb.unpack_tensor(mb.BitTensor(2, 40, 136, 64, tc.view(np.uint64)))
B = mb.unpack_tensor(mb.BitTensor(2, 40, 136, 64, gen.view(np.uint64)))
d = np.argwhere(A != B)
print("mismatches", len(d))
full = dense.ref_float_conv(x, w, b, 1, 1)
ts = mean - be * sigma / np.where(g == 0, 1.0, g)
S = np.abs(w).reshape(64, -1).sum(1)
for n, yy, xx, o in d[:20]:
    a = full[n, yy, xx, o]
    print(n, yy, xx, o, "tc", A[n, yy, xx, o], "gen", B[n, yy, xx, o], "acc", a, "T*", ts[o],
          "dist", a - ts[o], "rel to S", (a - ts[o]) / S[o], "g", g[o])
