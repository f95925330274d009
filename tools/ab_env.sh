#!/bin/bash
# A/B device timing of env-selected variants of the in-tree library:
#   tools/ab_env.sh "" "MBU_NBUF3=1" "MBU_COL_SPLIT=1" ...   ("" = defaults)
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu --no-cudnn --no-e2e --no-extra --steps 10 --warmup 5 > /dev/null 2>&1  # settle clocks
for envs in "$@"; do
  for rep in 1 2; do
    env $envs timeout 600 python bench.py --no-cpu --no-cudnn --no-e2e --no-extra --steps 20 --warmup 5 > gpurun_out/ab.json 2>gpurun_out/ab.err
    python - "${envs:-default}" <<'PY'
import json, sys
try:
    d = json.load(open("gpurun_out/ab.json"))
except Exception:
    print(sys.argv[1], "FAILED", open("gpurun_out/ab.err").read()[-800:]); raise SystemExit
ks = {k["layer"]: k["ms"] for k in d["kernel_breakdown"]}
print(f'{sys.argv[1]:28s} value {d["value"]:7.1f}  ' + " ".join(f'{n}={v:.3f}' for n, v in ks.items()))
PY
  done
done
