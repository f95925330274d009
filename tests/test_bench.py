"""bench.py keeps the driver's JSON contract (one line on rank 0)."""

from __future__ import annotations

import json
import subprocess
import sys

import pytest

from conftest import ROOT

COMMON = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
          "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"}


def _run(args, timeout):
    out = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                         timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"], 600)
    assert COMMON <= set(d) and d["impl"] == "reference"
    assert d["metric"] == "MBU-Net frames/s @1024x2048" and d["unit"] == "frames/s" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"


@pytest.mark.gpu
def test_our_arm_line():
    d = _run(["--steps", "3", "--warmup", "3", "--no-cpu", "--no-cudnn"], 900)
    assert COMMON - {"cpu_baseline"} <= set(d)
    assert {"roofline", "clocks", "gpu_launches"} <= set(d)
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] == "tensor" and 0 < r["frac"] < 1 and r["achieved"] > 0 and r["peak"] > 0
    assert d["gpu_launches"] > 0
    c2, c5 = d["config2_microbench"], d["config5_4k_latency"]
    assert all(r["exact_vs_oracle"] and r["fused_threshold_bits"]["tops"] > 0 for r in c2["rows"])
    assert c5["frames"] >= 200 and 0 < c5["device_ms"]["p50"] <= c5["device_ms"]["p99"]
