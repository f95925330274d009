#!/bin/bash
# up-CT1 256-column tiles + epilogue-halves barrier before tconv TMEM bias init
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bigshape.py tests/test_gpu_layers.py tests/test_gpu_forward.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for rep in 1 2; do
for envs in "" "MBU_TCONV_N128=1"; do
  env $envs timeout 600 python bench.py --no-cpu --no-cudnn --no-e2e --no-extra --steps 20 --warmup 5 > gpurun_out/ab.json 2>gpurun_out/ab.err
  python - "${envs:-n256}" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
ks = {k["layer"]: k["ms"] for k in d["kernel_breakdown"]}
print(f'{sys.argv[1]:24s} value {d["value"]:7.1f} ms {d["ms_per_step"]:.4f} CT1 {ks["up-CT1"]:.4f} CT2 {ks["up-CT2"]:.4f} CT3 {ks["up-CT3"]:.4f}')
PY
done; done
