#!/bin/bash
# A/B device timing of libraries: tools/ab_bench.sh lib1.so lib2.so ...  (default lib = in-tree)
mkdir -p gpurun_out
for lib in "$@"; do
  for rep in 1 2; do
    if [ "$lib" = default ]; then unset MBU_LIB; else export MBU_LIB=$lib; fi
    timeout 600 python bench.py --no-cpu --no-cudnn --no-e2e --steps 20 --warmup 5 > gpurun_out/ab.json 2>/dev/null
    python - "$lib" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
ks = {k["layer"]: k["ms"] for k in d["kernel_breakdown"]}
print(f'{sys.argv[1]:28s} value {d["value"]:7.1f}  ' + " ".join(f'{n}={v:.3f}' for n, v in ks.items()))
PY
  done
done
