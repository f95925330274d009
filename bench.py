#!/usr/bin/env python
"""MBU-Net forward throughput on B200 (BASELINE.json config 3 / 4).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one forward of a batch of 8 synthetic 3x1024x2048 float64 frames
through the default (all-masked) MBU-Net with random weights from the
activation-preserving generator. For N > 1 the driver launches this under
torchrun; each rank runs its own batch (replicas, frames sharded, no
collective on the data path — SURVEY.md §8(e)), so scaling is weak and the
reported value is frames of all ranks / max-over-ranks device time.

Rank 0 prints one JSON line. ``value`` is device-resident throughput (CUDA
graph replay, inputs already in HBM); ``e2e`` is the same metric through the
public engine with the image copied host->device from pinned memory and the
float64 logits + uint8 mask copied back every step. ``roofline`` is for the
dominant kernel (the tcgen05 conv), measured with CUDA events around every
layer of an eager forward. ``cpu_baseline`` times the reference CPU engine's
restatement (oracle/engine.py) on this host. ``cudnn_fp16`` is the paper's
comparison: a cuDNN FP16 U-Net of the same shape (baselines/cudnn_unet.py).

``--impl reference`` times the reference CPU path (the oracle port of the
packed engine, all host threads) on the same metric and config.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MBU-Net frames/s @1024x2048"
UNIT = "frames/s"
H, W, BATCH = 1024, 2048, 8
SEED = 0
# reference workload accounting (bitunet.planner.total_ops)
OPS_PER_FRAME = 1_933_809_025_024


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws <= 1:
        return None, 0, 1, 0
    import torch.distributed as dist

    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    return dist, rank, ws, local


def _config():
    import paper_2601_11660_b200 as mb

    return mb.UNetConfig(height=H, width=W)


def _model(cfg):
    import paper_2601_11660_b200 as mb

    return mb.build(cfg, mb.live_bundle(cfg, np.random.default_rng(SEED)))


def _frames(first: int) -> np.ndarray:
    """Frames first..first+BATCH-1 of the synthetic stream (quantizer.bench_frame)."""
    from paper_2601_11660_b200.quantizer import bench_frame

    return np.stack([bench_frame(first + i, H, W) for i in range(BATCH)])


def _cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------- CPU leg


def cpu_reference_step(model, image, threads=None):
    """One forward of ``image`` on the CPU port of the reference engine; returns seconds."""
    from oracle import engine as port

    threads = threads or _cores()
    t0 = time.perf_counter()
    port.forward(model, image, threads=threads)
    return time.perf_counter() - t0


def cpu_baseline(model):
    """The reference CPU path timed on ONE FULL 1024x2048 frame (bench frame 0)."""
    from paper_2601_11660_b200.quantizer import bench_frame

    cpu_reference_step(model, bench_frame(0, 256, 256)[None])  # warm-up (page-in, BLAS, OpenMP)
    t = cpu_reference_step(model, bench_frame(0, H, W)[None])
    return {
        "value": 1.0 / t,
        "unit": UNIT,
        "cores": _cores(),
        "kind": "port",
        "sample": f"1 full 1024x2048 frame (bench frame 0), no scaling: oracle/engine.py packed "
                  f"XOR-popcount engine (im2row + oracle/xorpop.c rows), {_cores()} threads on "
                  f"{_cpu_model()}",
        "seconds_per_frame": t,
    }


def cpu_numba_baseline(cfg, sample=(512, 512)):
    """bitunet's own Numba forward, if the unmodified reference
    is installed in baseline/_ref (tools/install_reference.sh). A bounded sample:
    one 512x512 frame; reported per pixel-scaled 1024x2048 frame and as measured."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "bitunet").is_dir():
        return {"unavailable": "baseline/_ref not installed"}
    code = f"""
import json, os, sys, time
import numpy as np
sys.path[:0] = [{str(ref)!r}, {str(ROOT)!r}]
import bitunet as R
from paper_2601_11660_b200 import quantizer as Q
from paper_2601_11660_b200.quantizer import bench_frame
cfg = R.UNetConfig(height={sample[0]}, width={sample[1]})
mine = Q.live_bundle(R.UNetConfig(height={H}, width={W}), np.random.default_rng({SEED}))
rb = R.WeightBundle()
for name, e in mine.entries.items():
    rb.add(R.BundleEntry(name, e.kind, e.weights, bias=e.bias, gamma=e.gamma, beta=e.beta,
                         mean=e.mean, var=e.var, eps=e.eps))
model = R.build(cfg, rb)
img = bench_frame(0, {sample[0]}, {sample[1]})[None]
thr = len(os.sched_getaffinity(0))
small = R.build(R.UNetConfig(height=64, width=64), rb)  # warm-up: Numba JIT, thread pool
R.forward(small, bench_frame(1, 64, 64)[None], threads=thr)
t0 = time.perf_counter()
R.forward(model, img, threads=thr)
print(json.dumps({{"seconds": time.perf_counter() - t0, "threads": thr}}))
"""
    env = dict(os.environ, NUMBA_CACHE_DIR=os.environ.get("NUMBA_CACHE_DIR", "/tmp/mbu_numba_cache"),
               PYTHONDONTWRITEBYTECODE="1", MBU_REFERENCE_ERRORS="0")
    try:
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                           timeout=600)
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001 - a reported baseline only
        return {"unavailable": f"bitunet forward failed: {type(e).__name__}"}
    scale = (H * W) / (sample[0] * sample[1])
    return {
        "value": 1.0 / (d["seconds"] * scale), "unit": UNIT, "cores": d["threads"],
        "kind": "reference",
        "sample": f"bitunet 0.1.0 graph.forward (Numba JIT path, unmodified, baseline/_ref), one "
                  f"{sample[0]}x{sample[1]} frame measured in {d['seconds']:.2f} s with "
                  f"threads={d['threads']}; value = that time scaled by pixel count x{scale:g} to a "
                  f"1024x2048 frame (the network's cost is linear in pixels)",
        "seconds_per_sample": d["seconds"],
    }


def run_reference(args):
    """The reference arm: the CPU port of the reference engine on the box's host
    cores, one FULL 1024x2048 frame per step (no scaling). value = frames / time."""
    from paper_2601_11660_b200.quantizer import bench_frame

    dist, rank, world, local = _dist()
    if rank != 0:
        return 0
    cfg = _config()
    model = _model(cfg)
    warm = bench_frame(0, 512, 512)[None]
    for _ in range(args.warmup):  # untimed warm-up on a 512x512 frame (page-in, OpenMP pool)
        cpu_reference_step(model, warm)
    times = [cpu_reference_step(model, bench_frame(i % BATCH, H, W)[None]) for i in range(args.steps)]
    total = sum(times)
    value = args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64 bitplanes / int32 acc / f64 endpoints",
        "data": "synthetic: live-generator random weights (seed 0), bench_frame images",
        "config": {"workload": "MBU-Net forward, 3x1024x2048 frames (config 3); one step = one "
                               "full frame of the batch-8 stream", "global_batch": BATCH,
                   "height": H, "width": W, "parallelism": "cpu", "frames_per_step": 1},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": _cores(), "kind": "port",
                         "sample": f"each timed step = 1 full 1024x2048 frame (no scaling), "
                                   f"oracle/engine.py, {_cores()} threads, {_cpu_model()}; "
                                   f"warm-up steps on a 512x512 frame"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- clocks


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(gpu_index), "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        rows = []
        for line in out.splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), float(parts[2]), parts[3:]))
            except ValueError:
                continue
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        loaded = [r for r in rows if r[2] > 250.0] or rows
        reasons = sorted({names[i] for r in loaded for i, v in enumerate(r[3]) if v == "Active"})
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": rows[0][1],
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(loaded),
                "power_w_max": max(r[2] for r in rows)}


# ----------------------------------------------------------------- GPU leg


def layer_ops(model, n):
    """Algorithmic ops (2*MAC, real K) of every layer (planner._entry_ops)."""
    ops = []
    h, w = H, W
    for layer in model.layers:
        s = layer.spec
        if layer.kind == "maxpool":
            h, w = h // 2, w // 2
            ops.append(0)
        elif layer.kind == "concat":
            ops.append(0)
        elif layer.kind.endswith("tconv"):
            h, w = h * s.stride, w * s.stride
            ops.append(2 * n * h * w * s.c_out * s.c_in)
        else:
            h = (h + 2 * s.padding - s.kernel_h) // s.stride + 1
            w = (w + 2 * s.padding - s.kernel_w) // s.stride + 1
            ops.append(2 * n * h * w * s.c_out * s.c_in * s.kernel_h * s.kernel_w)
    return ops


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def _profile_traffic():
    p = ROOT / "profiles" / "ncu_conv_tc_summary.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("dram_bytes_per_launch_avg")
        except (ValueError, OSError):
            return None
    return None


# ----------------------------------------------------------------- configs 2 and 5

C2_OPS = 19_327_352_832  # 2 * 128 * 128 * 256 * (9 * 256): SURVEY.md 8(d), config 2


def config2_microbench(dev, reps=200):
    """BASELINE config 2: one masked 3x3 conv, 256 -> 256 channels, 1 x 128 x 128, at
    50 / 90 / 95 % weight sparsity (ternary weights, P(0) = s, non-zeros +-1).
    Device time of the tcgen05 conv per call (CUDA events around a CUDA graph of
    `reps` launches), once producing the reference's int32 accumulators
    (conv_forward, layers.py:289-313) and once with the fused threshold + packed
    bits the network runs; checked exactly against the CPU oracle first."""
    import torch

    import paper_2601_11660_b200 as mb
    from oracle import engine as port
    from paper_2601_11660_b200.ops import ConvHandle, _words_to_dev

    rng = np.random.default_rng(0)
    acts = (rng.integers(0, 2, (1, 128, 128, 256)) * 2 - 1).astype(np.int8)
    x = mb.pack_tensor(acts)
    spec = mb.ConvSpec(3, 3, 1, 1, 256, 256)
    rows = []
    xd = _words_to_dev(x.words, dev)
    for sp in (0.5, 0.9, 0.95):
        nz = rng.random((256, 3, 3, 256)) >= sp
        w = np.where(nz, rng.choice((-1, 1), size=nz.shape), 0).astype(np.int8)
        planes = mb.pack_conv_weights(w, x.segments, masked=True)
        thr = mb.FusedThreshold(np.zeros(256, np.int32), np.zeros(256, np.uint8))
        cv = ConvHandle(planes, spec, x.segments, thr, device=dev)
        acc = torch.empty((1, 128, 128, 256), dtype=torch.int32, device=dev)
        bits = torch.empty((1, 128, 128, cv.out_wpp), dtype=torch.int64, device=dev)
        cv.run(xd, 1, 128, 128, acc=acc)
        torch.cuda.synchronize(dev)
        want = port.conv_forward(x.words, [(g.lane_offset, g.count) for g in x.segments], planes, spec, 8)
        exact = bool(np.array_equal(acc.cpu().numpy(), want))
        res = {"sparsity": sp, "exact_vs_oracle": exact}
        for name, kw in (("acc_int32", {"acc": acc}), ("fused_threshold_bits", {"bits": bits})):
            st = torch.cuda.Stream(dev)
            with torch.cuda.stream(st):
                for _ in range(3):
                    cv.run(xd, 1, 128, 128, **kw)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st):
                    for _ in range(reps):
                        cv.run(xd, 1, 128, 128, **kw)
            times = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(st):  # (replay runs on the current stream)
                    e0.record(st)
                    g.replay()
                    e1.record(st)
                torch.cuda.synchronize(dev)
                times.append(e0.elapsed_time(e1) / reps)
            ms = statistics.median(times)
            res[name] = {"us_per_conv": 1e3 * ms, "tops": C2_OPS / (ms / 1e3) / 1e12}
        rows.append(res)
    return {"workload": "config 2: masked 3x3 conv 256->256, 1x128x128, ternary weights",
            "ops_per_conv": C2_OPS, "rows": rows,
            "how": "CUDA graph of 200 back-to-back launches of the tcgen05 conv (ConvHandle.run), "
                   "median of 5 replays; 16384 output pixels fill 128 of 148 SMs once, so this is a "
                   "latency-bound size for one GPU"}


def config2_reference_cpu():
    """The reference's own micro_bench (bitunet.bench.micro_bench, bench.py:207-243) at
    config 2's shape on this host, from the unmodified install in baseline/_ref."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "bitunet").is_dir():
        return {"unavailable": "baseline/_ref not installed"}
    code = f"""
import json, os, sys
sys.path.insert(0, {str(ref)!r})
from bitunet.bench import micro_bench
thr = len(os.sched_getaffinity(0))
mb = micro_bench(channels=256, extent=128, kernel=3, reps=3, threads=thr, include_oracle=False)
print(json.dumps({{"seconds": mb.t_bit, "threads": thr, "n_ops": mb.n_ops}}))
"""
    env = dict(os.environ, NUMBA_CACHE_DIR=os.environ.get("NUMBA_CACHE_DIR", "/tmp/mbu_numba_cache"),
               PYTHONDONTWRITEBYTECODE="1", MBU_REFERENCE_ERRORS="0")
    try:
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600)
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001 - a reported baseline only
        return {"unavailable": f"micro_bench failed: {type(e).__name__}"}
    return {"seconds_per_conv": d["seconds"], "gops": d["n_ops"] / d["seconds"] / 1e9, "threads": d["threads"],
            "what": "bitunet.bench.micro_bench(channels=256, extent=128) conv_forward time (its own "
                    "uniform ternary weights), Numba XOR-popcount path, all host threads"}


def config5_latency(dev, frames=200):
    """BASELINE config 5: 4K (3x2160x3840) batch-1 per-frame latency, p50/p99 over
    `frames` frames: device (CUDA-graph replay, image resident) and end to end
    (pinned float64 frame H2D + forward + uint8 mask and float64 logits D2H, one
    stream, synchronised per frame)."""
    import torch

    import paper_2601_11660_b200 as mb
    from paper_2601_11660_b200.quantizer import bench_frame

    cfg = mb.UNetConfig(height=2160, width=3840)
    model = mb.build(cfg, mb.live_bundle(cfg, np.random.default_rng(SEED)))
    eng = mb.Engine(model, batch=1, device=dev)
    host = torch.from_numpy(bench_frame(0, 2160, 3840)[None]).pin_memory()
    hl = torch.empty(eng.out_shape, dtype=torch.float64, pin_memory=True)
    hm = torch.empty(eng.out_shape, dtype=torch.uint8, pin_memory=True)
    eng.image.copy_(host)
    for _ in range(10):
        eng.run()
    torch.cuda.synchronize(dev)

    def pct(v, q):
        v = sorted(v)
        return v[min(len(v) - 1, int(round(q * (len(v) - 1))))]

    dev_ms, e2e_ms = [], []
    for _ in range(frames):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(eng.stream)
        eng.run()
        e1.record(eng.stream)
        e1.synchronize()
        dev_ms.append(e0.elapsed_time(e1))
    for _ in range(frames):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(eng.stream)
        eng.run_e2e(host, hl, hm)
        e1.record(eng.stream)
        e1.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    ops = 7_648_365_772_800
    out = {"workload": "config 5: MBU-Net 1x3x2160x3840, batch 1", "frames": frames,
           "device_ms": {"p50": pct(dev_ms, 0.5), "p99": pct(dev_ms, 0.99), "min": min(dev_ms)},
           "e2e_ms": {"p50": pct(e2e_ms, 0.5), "p99": pct(e2e_ms, 0.99), "min": min(e2e_ms)},
           "device_tops_p50": ops / (pct(dev_ms, 0.5) / 1e3) / 1e12,
           "h2d_bytes_per_frame": host.numel() * 8, "d2h_bytes_per_frame": hl.numel() * 8 + hm.numel(),
           "how": "Engine (CUDA graph), CUDA events per frame on the engine stream; e2e = run_e2e "
                  "(pinned image H2D, replay, logits + mask D2H) synchronised per frame"}
    del eng
    torch.cuda.empty_cache()
    return out


STREAM = 64  # config 4: a 64-frame stream over the node's GPUs


def run_multi(args):
    """BASELINE config 4 (N > 1): a 64-frame 1024x2048 stream sharded contiguously
    over the N ranks (dp.StreamRunner: 64/N frames each, batches of 8, no
    collective on the data path), strong scaling. ``value``: device-resident
    forwards of every rank's shard; ``e2e``: pinned 8-bit frames H2D, GPU decode,
    forward, GPU-packed masks, and the final gather of all packed masks to rank 0
    (NCCL) plus its D2H. Both timed on the device, max over ranks."""
    import torch

    import paper_2601_11660_b200 as mb
    from paper_2601_11660_b200 import _lib, dp

    dist, rank, world, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    cfg = _config()
    model = _model(cfg)
    runner = dp.StreamRunner(model, STREAM, batch=BATCH, dist=dist, device=dev)
    eng = runner.engine
    eng.image.copy_(torch.from_numpy(_frames(runner.lo)))

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    clocks = ClockSampler(local)
    for _ in range(args.warmup):
        runner.run_resident()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    before = _lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(eng.stream)
    for _ in range(args.steps):
        runner.run_resident()
    e1.record(eng.stream)
    torch.cuda.synchronize()
    launches = _lib.launch_count() - before
    dist.barrier()
    dev_ms = max_over_ranks(e0.elapsed_time(e1))
    value = STREAM * args.steps / (dev_ms / 1e3)

    e2e = None
    if not args.no_e2e:
        g = torch.Generator().manual_seed(77 + rank)
        raster = torch.randint(0, 256, (runner.n_local, H, W, 3), dtype=torch.uint8, generator=g).pin_memory()
        for _ in range(args.warmup):
            runner.run(raster)
            runner.gather(0)
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        eng._ensure_slots()
        h0.record(eng.h2d)
        for _ in range(args.steps):
            runner.run(raster)
            runner.gather(0)
        h1.record(torch.cuda.current_stream(dev))
        torch.cuda.synchronize()
        dist.barrier()
        e2e_ms = max_over_ranks(h0.elapsed_time(h1))
        e2e = {"value": STREAM * args.steps / (e2e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": STREAM * H * W * 3,
               "d2h_bytes_per_step": STREAM * ((H * W + 7) // 8),
               "ms_per_step": e2e_ms / args.steps,
               "how": "dp.StreamRunner per rank: pinned 8-bit frames H2D (copy stream), "
                      "decode_raster + CUDA-graph forward + pack_mask_bits on the GPU, then "
                      "gather of every rank's bit-packed masks to rank 0 (NCCL) and D2H there"}
    clk = clocks.stop()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "e2m1 (tcgen05 kind::mxf4, exact f32 integer acc) 3x3 convs / s8 tconvs / "
                     "u64 bitplanes / f64 endpoints",
            "data": "synthetic: live-generator random weights (seed 0), bench_frame images "
                    "(resident), random 8-bit frames (e2e)",
            "config": {"workload": f"config 4: MBU-Net 64-frame 3x1024x2048 stream over {world} GPUs "
                                   f"({STREAM // world} frames each, batches of {BATCH})",
                       "global_batch": STREAM, "height": H, "width": W,
                       "parallelism": f"dp{world} (frame shards, no data-path collective)",
                       "l2": "inputs and activations larger than L2"},
            "e2e": e2e, "roofline": None, "cpu_baseline": None, "clocks": clk,
            "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


def run_ours(args):
    import torch

    import paper_2601_11660_b200 as mb
    from paper_2601_11660_b200 import _lib

    dist, rank, world, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if dist is not None:
        dist.init_process_group("nccl", device_id=dev)
    cfg = _config()
    model = _model(cfg)
    eng = mb.Engine(model, batch=BATCH, device=dev)
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    # the benchmark stream's frames (rank r runs frames 8r..8r+7); frames 0 and
    # 7 are parity-pinned against the reference (tests/test_gpu_bigshape.py)
    eng.image.copy_(torch.from_numpy(_frames(rank * BATCH)))
    st = eng.stream

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    clocks = ClockSampler(local)
    # ---- device-resident throughput (graph replay)
    for _ in range(args.warmup):
        eng.run()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.steps):
        eng.run()
    e1.record(st)
    torch.cuda.synchronize()
    barrier()
    dev_ms = max_over_ranks(e0.elapsed_time(e1))
    value = world * BATCH * args.steps / (dev_ms / 1e3)

    # ---- end to end through the public engine: pinned H2D + forward + D2H
    e2e = None
    if not args.no_e2e:
        # two distinct pinned host frames batches, two result buffers
        host_imgs = []
        for i in range(2):
            hb = torch.empty(eng.shape, dtype=torch.float64, pin_memory=True)
            hb.copy_(torch.from_numpy(_frames((2 * rank + i) * BATCH)))
            host_imgs.append(hb)
        host_logits = [torch.empty(eng.out_shape, dtype=torch.float64, pin_memory=True) for _ in range(2)]
        host_masks = [torch.empty(eng.out_shape, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        eng.run_stream(host_imgs, host_logits, host_masks, args.warmup)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        e0.record(eng.h2d)
        eng.run_stream(host_imgs, host_logits, host_masks, args.steps)
        e1.record(eng.d2h)
        torch.cuda.synchronize()
        barrier()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1))
        e2e = {"value": world * BATCH * args.steps / (e2e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": host_imgs[0].numel() * 8,
               "d2h_bytes_per_step": host_logits[0].numel() * 8 + host_masks[0].numel(),
               "ms_per_step": e2e_ms / args.steps,
               "how": "Engine.run_stream: pinned float64 images H2D on a copy stream, CUDA-graph "
                      "forward, float64 logits + uint8 mask D2H on a second copy stream; two "
                      "device buffer sets overlap step i's compute with i+1's upload / i-1's "
                      "download"}
        # same loop fed with 8-bit netpbm samples, decoded on the GPU (decode_raster)
        host_r = [torch.empty(eng.shape, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        for hr in host_r:
            hr.copy_(torch.randint(0, 256, eng.shape, dtype=torch.uint8, device=dev, generator=g).cpu())
        eng.run_stream_raster(host_r, 255, host_logits, host_masks, args.warmup)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        e0.record(eng.h2d)
        eng.run_stream_raster(host_r, 255, host_logits, host_masks, args.steps)
        e1.record(eng.d2h)
        torch.cuda.synchronize()
        barrier()
        r_ms = max_over_ranks(e0.elapsed_time(e1))
        e2e["raster_u8"] = {
            "value": world * BATCH * args.steps / (r_ms / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": host_r[0].numel(),
            "d2h_bytes_per_step": host_logits[0].numel() * 8 + host_masks[0].numel(),
            "ms_per_step": r_ms / args.steps,
            "how": "Engine.run_stream_raster: pinned 8-bit P6 samples H2D, mbu_decode_raster "
                   "(sample/255, bit-identical to read_image) + forward, same D2H"}
    clk = clocks.stop()

    line = None
    if rank == 0:
        # ---- per-layer CUDA-event timing of eager forwards (roofline)
        dm = eng.dm
        dm.set_timing(True)
        reps = 3
        acc_t = None
        for _ in range(reps):
            with torch.cuda.stream(st):
                # keep the GPU busy while the host enqueues the eager forward, so no
                # layer's events include host launch latency (tensor-map encodes etc.)
                torch.cuda._sleep(4_000_000)
                eng._enqueue()
            t = dm.layer_times()
            acc_t = t if acc_t is None else [a + b for a, b in zip(acc_t, t)]
        dm.set_timing(False)
        lt = [x / reps for x in acc_t]
        ops = layer_ops(model, BATCH)
        # dominant kernel: the 3x3 binary convs (conv_tc_kernel<9>, tcgen05 kind::mxf4 with
        # e2m1 operands, 17 launches per step); the 2x2/s2 tconvs run kind::i8 (4 launches)
        fp4 = not os.environ.get("MBU_CONV_I8")
        is3 = [("conv" in l.kind and l.kind != "float-conv" and "tconv" not in l.kind) for l in model.layers]
        c3_ops = sum(o for o, k in zip(ops, is3) if k)
        c3_ms = sum(t for t, k in zip(lt, is3) if k)
        step_ms = sum(lt)
        peaks, src = _peaks()
        # burst figure: the step runs at the maximum SM clock, far under the power cap
        # (clocks.sm_mhz / power_w_max below), which is what the sustained figure models
        bf16 = peaks["bf16_tflops"]
        peak = (4.0 if fp4 else 2.0) * bf16
        achieved = c3_ops / (c3_ms / 1e3) / 1e12
        # the e2m1 MMA rate measured by tools/ubench_fp4.cu (16368 MAC/clk/SM) at the max clock
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        ubench_peak = 16368 * 2 * sms * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        breakdown = [
            {"layer": l.name, "kind": l.kind, "ms": round(t, 4),
             "tops": round(o / (t / 1e3) / 1e12, 1) if o and t > 0 else None}
            for l, t, o in zip(model.layers, lt, ops) if l.kind != "concat"]
        # MBU_FUSED_HEAD=1: the 1x1 head runs inside the epilogue of the conv before it
        # (no launch of its own); its row then times only the empty event pair
        if os.environ.get("MBU_FUSED_HEAD") and eng.launches_per_run == sum(
                l.kind != "concat" for l in model.layers) - 1:
            breakdown[-1]["fused_into"] = breakdown[-2]["layer"] + " epilogue (its ms include the head)"
            breakdown[-1]["tops"] = None
        roofline = {
            "bound": "tensor",
            "kernel": ("conv_tc_kernel<9> 3x3 binary convs (tcgen05.mma kind::mxf4, e2m1 "
                       "{-1,0,+1} x {0,1}, exact f32 integer accumulation)" if fp4 else
                       "conv_tc_kernel<9> 3x3 binary convs (tcgen05.mma kind::i8)"),
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": _profile_traffic(),
            "peak_source": (f"{'4' if fp4 else '2'} x bf16_tflops (burst) of {src} MEASURED_PEAKS.json "
                            f"(sm_100 dense {'FP4' if fp4 else 'int8'} rate = {'4' if fp4 else '2'}x bf16)"),
            "peak_mma_ubench": ubench_peak,
            "frac_of_mma_ubench": achieved / ubench_peak,
            "peak_mma_ubench_source": "tools/ubench_fp4.cu: 16368 e2m1 MAC/clk/SM (kind::mxf4, N >= 128) "
                                      "x 2 x SMs x sm_max_mhz",
            "ops_per_launch_basis": "2*MAC with the reference's real K (planner.total_ops) summed over "
                                    "the 17 3x3 conv launches of one step, over their summed CUDA-event time",
            "share_of_step": c3_ms / step_ms,
            "launches": int(sum(is3)),
        }
        cudnn = None
        if not args.no_cudnn and world == 1:
            from baselines.cudnn_unet import CudnnUNetRunner

            runner = CudnnUNetRunner(cfg, BATCH, dev)
            for _ in range(args.warmup):
                runner.run()
            torch.cuda.synchronize()
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(runner.stream)
            for _ in range(args.steps):
                runner.run()
            c1.record(runner.stream)
            torch.cuda.synchronize()
            cms = c0.elapsed_time(c1) / args.steps
            cudnn = {"value": BATCH / (cms / 1e3), "unit": UNIT, "ms_per_step": cms,
                     "what": "cuDNN FP16 U-Net, same channel schedule, channels_last, "
                             "cudnn.benchmark, CUDA graph (baselines/cudnn_unet.py)",
                     "speedup_ours_vs_cudnn": (BATCH * args.steps / (dev_ms / 1e3)) / (BATCH / (cms / 1e3))}
            del runner
            torch.cuda.empty_cache()
            try:  # the fused (torch.compile'd) FP16 baseline: bias/ReLU/concat fused around cuDNN
                runner = CudnnUNetRunner(cfg, BATCH, dev, fused=True)
                for _ in range(args.warmup):
                    runner.run()
                torch.cuda.synchronize()
                c0.record(runner.stream)
                for _ in range(args.steps):
                    runner.run()
                c1.record(runner.stream)
                torch.cuda.synchronize()
                fms = c0.elapsed_time(c1) / args.steps
                cudnn["fused"] = {"value": BATCH / (fms / 1e3), "unit": UNIT, "ms_per_step": fms,
                                  "what": "same FP16 U-Net through torch.compile (Inductor: cuDNN "
                                          "convs, fused bias/ReLU/concat), CUDA graph",
                                  "speedup_ours_vs_fused": (BATCH * args.steps / (dev_ms / 1e3)) / (BATCH / (fms / 1e3))}
                del runner
            except Exception as e:  # noqa: BLE001 - a reported baseline only
                cudnn["fused"] = {"unavailable": f"{type(e).__name__}: {str(e)[:200]}"}
            torch.cuda.empty_cache()
        cpu = numba = None
        if not args.no_cpu and world == 1:
            cpu = cpu_baseline(model)
            numba = cpu_numba_baseline(cfg)
        c2 = c5 = api = None
        if not args.no_extra and world == 1:
            try:  # the drop-in reference API: numpy float64 batch in, numpy logits + mask out
                imgs = _frames(0)
                mb.forward(model, imgs, device=dev)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for _ in range(3):
                    mb.forward(model, imgs, device=dev)
                ta = (time.perf_counter() - t0) / 3
                api = {"value": BATCH / ta, "unit": UNIT, "ms_per_batch": 1e3 * ta,
                       "what": "paper_2601_11660_b200.forward(model, numpy (8,1024,2048,3) float64) -> "
                               "ForwardResult with numpy float64 logits + uint8 mask: the reference's "
                               "graph.forward contract (host arrays in and out, synchronous), host wall "
                               "clock per call including the 403 MB upload (chunked through a cached "
                               "page-locked staging buffer) and the 151 MB download (DMA into a cached "
                               "page-locked buffer, then a host copy into ordinary numpy arrays)"}
                del imgs
            except Exception as e:  # noqa: BLE001
                api = {"error": f"{type(e).__name__}: {str(e)[:200]}"}
            try:
                c2 = config2_microbench(dev)
                if not args.no_cpu:
                    c2["reference_cpu"] = config2_reference_cpu()
            except Exception as e:  # noqa: BLE001 - extra keys must not sink the headline line
                c2 = {"error": f"{type(e).__name__}: {str(e)[:200]}"}
            try:
                c5 = config5_latency(dev)
            except Exception as e:  # noqa: BLE001
                c5 = {"error": f"{type(e).__name__}: {str(e)[:200]}"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dev_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None,
            "dtype": "e2m1 (tcgen05 kind::mxf4, exact f32 integer acc) 3x3 convs / s8 (kind::i8, s32 acc) "
                     "tconvs / u64 bitplanes / f64 endpoints",
            "data": "synthetic: live-generator random weights (seed 0), uniform [0,1) float64 images",
            "config": {"workload": "MBU-Net forward, batch 8 per GPU, 3x1024x2048 (config 3; "
                                   "config 4 when N>1)", "global_batch": BATCH * world,
                       "height": H, "width": W, "parallelism": f"dp{world} (replicas)",
                       "l2": "inputs and activations larger than L2 (403 MB image per step)"},
            "e2e": e2e,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "cpu_baseline_bitunet_numba": numba,
            "cudnn_fp16": cudnn,
            "clocks": clk,
            "gpu_launches": eng.launches_per_run * args.steps,
            "kernel_breakdown": breakdown,
            "api_forward": api,
            "config2_microbench": c2,
            "config5_4k_latency": c5,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cudnn", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the config 2 / config 5 keys")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        return run_multi(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
