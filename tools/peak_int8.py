"""Measure dense tensor-core peaks on this B200 (cuBLAS int8 and bf16), CUDA events.

    python tools/peak_int8.py  -> one JSON line
"""
import json

import torch


def timed(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters / 1e3


out = {}
for n in (8192, 16384):
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t()
    t = timed(lambda: torch._int_mm(a, b), 20)
    out[f"int8_tops_{n}"] = 2 * n**3 / t / 1e12
    x = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
    y = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
    t = timed(lambda: x @ y, 20)
    out[f"bf16_tflops_{n}"] = 2 * n**3 / t / 1e12
# sustained: a ~5 s loop
n = 8192
a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t()
t = timed(lambda: torch._int_mm(a, b), 2000)
out["int8_tops_sustained_8192"] = 2 * n**3 / t / 1e12
print(json.dumps(out))
