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
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
