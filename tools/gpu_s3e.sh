#!/bin/bash
# stem early accumulator release: stem/forward parity tests + A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layers.py tests/test_gpu_forward.py tests/test_gpu_bigshape.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for rep in 1 2; do
for envs in "" "MBU_STEM_LATE_RELEASE=1"; do
  env $envs timeout 600 python bench.py --no-cpu --no-cudnn --no-e2e --no-extra --steps 20 --warmup 5 > gpurun_out/ab.json 2>gpurun_out/ab.err
  python - "${envs:-early}" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
ks = {k["layer"]: k["ms"] for k in d["kernel_breakdown"]}
print(f'{sys.argv[1]:24s} value {d["value"]:7.1f} ms {d["ms_per_step"]:.4f} stem {ks["stem"]:.4f}')
PY
done; done
