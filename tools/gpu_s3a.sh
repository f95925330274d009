#!/bin/bash
# fused head: GPU tests, device bench with and without the fusion (A/B)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for rep in 1 2; do
for envs in "" "MBU_UNFUSED_HEAD=1"; do
  env $envs timeout 600 python bench.py --no-cpu --no-cudnn --no-e2e --no-extra --steps 20 --warmup 5 > gpurun_out/ab.json 2>gpurun_out/ab.err
  python - "${envs:-fused}" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
ks = {k["layer"]: k["ms"] for k in d["kernel_breakdown"]}
print(f'{sys.argv[1]:20s} value {d["value"]:7.1f} frac {d["roofline"]["frac"]:.3f} launches {d.get("gpu_launches")} upC4b {ks["up-C4.b"]:.4f} head {ks["head"]:.4f}')
PY
done; done
