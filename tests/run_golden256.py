"""Config-1 (256x256) golden check in a fresh process, so that build-time
environment switches of the engine (MBU_PAIR, MBU_SB64, ... read once per
process) can be exercised: every layer's packed words and accumulators must
match the reference's per-layer SHA-256 digests, the mask exactly, the
logits within 1e-9. usage: python tests/run_golden256.py <gen> <seed>"""
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parent))

import numpy as np  # noqa: E402

import paper_2601_11660_b200 as mb  # noqa: E402
from conftest import load_golden  # noqa: E402
from test_gpu_forward import FLOAT_TOL, sha  # noqa: E402
from tests_golden_models import golden_model_256  # noqa: E402

gen, seed = sys.argv[1], int(sys.argv[2])
z = load_golden("forward_256.npz")
key = f"{gen}{seed}@256"
cfg, bundle, model, image = golden_model_256(gen, seed)
res = mb.forward(model, image, trace=True)
assert np.allclose(res.logits, z[f"{key}/logits"], rtol=FLOAT_TOL, atol=FLOAT_TOL)
assert np.array_equal(res.mask, z[f"{key}/mask"])
n = 0
for layer in model.layers:
    rec = res.trace[layer.name]
    k_out, k_acc = f"{key}/{layer.name}/out_sha", f"{key}/{layer.name}/acc_sha"
    if k_out in z.files:
        assert sha(rec["out"].words) == bytes(z[k_out]).decode(), layer.name
        n += 1
    if k_acc in z.files:
        assert sha(rec["acc"]) == bytes(z[k_acc]).decode(), layer.name
        n += 1
# the untraced forward (the benchmark's epilogue paths) must give the same mask
res2 = mb.forward(model, image)
assert np.array_equal(res2.mask, res.mask) and np.array_equal(res2.logits, res.logits)
print(f"golden256 {key} ok ({n} digests)")
