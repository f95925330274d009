import torch, time
dev = torch.device("cuda", 0)
n = 403 * 1024 * 1024 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device=dev)
o_d = torch.empty(151 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
o_h = torch.empty_like(o_d, device="cpu").pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for mode in ("h2d", "h2d+d2h", "h2d_chunks4"):
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(s1)
        with torch.cuda.stream(s1):
            for _ in range(5):
                if mode == "h2d_chunks4":
                    for c in range(4):
                        d[c * n // 4:(c + 1) * n // 4].copy_(h[c * n // 4:(c + 1) * n // 4], non_blocking=True)
                else:
                    d.copy_(h, non_blocking=True)
        if mode == "h2d+d2h":
            with torch.cuda.stream(s2):
                for _ in range(5):
                    o_h.copy_(o_d, non_blocking=True)
        e1.record(s1)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(mode, f"{5 * n * 8 / (ms / 1e3) / 1e9:.1f} GB/s H2D")
