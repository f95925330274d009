"""Wall-clock of the drop-in forward() (numpy in, numpy out) at the bench workload."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2601_11660_b200 as mb  # noqa: E402
from paper_2601_11660_b200.quantizer import bench_frame  # noqa: E402

cfg = mb.UNetConfig(height=1024, width=2048)
model = mb.build(cfg, mb.live_bundle(cfg, np.random.default_rng(0)))
imgs = np.stack([bench_frame(i, 1024, 2048) for i in range(8)])
r0 = mb.forward(model, imgs, device="cuda:0")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    r = mb.forward(model, imgs, device="cuda:0")
dt = (time.perf_counter() - t0) / 5
print(f"forward(): {1e3 * dt:.1f} ms per batch of 8 -> {8 / dt:.1f} frames/s; "
      f"same result: {np.array_equal(r.mask, r0.mask) and np.array_equal(r.logits, r0.logits)}")

# where the time goes
from paper_2601_11660_b200 import runtime as rt  # noqa: E402

dev = torch.device("cuda:0")
print("torch threads", torch.get_num_threads())
for name, fn in [
    ("np.ascontiguousarray", lambda: np.ascontiguousarray(imgs)),
    ("upload (staged)", lambda: rt._upload(imgs, dev)),
    ("upload (pageable .to)", lambda: torch.from_numpy(imgs).to(dev)),
]:
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    print(f"{name}: {1e3 * (time.perf_counter() - t0) / 3:.1f} ms")
src = torch.from_numpy(imgs).reshape(-1)
stage = torch.empty(src.numel(), dtype=torch.float64, pin_memory=True)
t0 = time.perf_counter()
for _ in range(3):
    stage.copy_(src)
print(f"host copy into pinned: {1e3 * (time.perf_counter() - t0) / 3:.1f} ms")
d = torch.empty(src.numel(), dtype=torch.float64, device=dev)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    d.copy_(stage, non_blocking=True)
torch.cuda.synchronize()
print(f"pinned H2D: {1e3 * (time.perf_counter() - t0) / 3:.1f} ms")
lg = torch.empty((8, 1024, 2048, 1), dtype=torch.float64, device=dev)
for name, fn in [("download pinned", lambda: (rt._download(lg), torch.cuda.synchronize())),
                 ("download .cpu()", lambda: lg.cpu())]:
    fn()
    t0 = time.perf_counter()
    for _ in range(3):
        fn()
    print(f"{name} (134 MB): {1e3 * (time.perf_counter() - t0) / 3:.1f} ms")
