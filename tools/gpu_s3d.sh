#!/bin/bash
# nibble head default: full GPU suite, A/B fused (nibble epilogue) vs head kernel vs byte-table head
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for rep in 1 2; do
for envs in "" "MBU_FUSED_HEAD=1" "MBU_HEAD_BYTETAB=1"; do
  env $envs timeout 600 python bench.py --no-cpu --no-cudnn --no-e2e --no-extra --steps 20 --warmup 5 > gpurun_out/ab.json 2>gpurun_out/ab.err
  python - "${envs:-nibble}" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
ks = {k["layer"]: k["ms"] for k in d["kernel_breakdown"]}
print(f'{sys.argv[1]:24s} value {d["value"]:7.1f} ms {d["ms_per_step"]:.4f} head {ks["head"]:.4f} upC4b {ks["up-C4.b"]:.4f}')
PY
done; done
