#!/bin/bash
# interleaved A/B of libraries on the stem (and the value), 3 reps each
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu --no-cudnn --no-e2e --no-extra --steps 10 --warmup 5 > /dev/null 2>&1
for rep in 1 2 3; do
  for lib in "$@"; do
    MBU_LIB=$lib timeout 600 python bench.py --no-cpu --no-cudnn --no-e2e --no-extra --steps 20 --warmup 5 > gpurun_out/ab.json 2>gpurun_out/ab.err
    python - "$lib" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
ks = {k["layer"]: k["ms"] for k in d["kernel_breakdown"]}
print(f'{sys.argv[1]:24s} value {d["value"]:7.1f} stem {ks["stem"]:.3f} stem2 {ks["stem2"]:.3f} upC4a {ks["up-C4.a"]:.3f} sum {sum(ks.values()):.3f}')
PY
  done
done
