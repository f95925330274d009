#!/bin/bash
# head kernels: nibble-table variant parity (vs reference goldens) + A/B + ncu full captures
mkdir -p gpurun_out
MBU_HEAD_NIB=1 timeout 900 python -m pytest tests/test_gpu_forward.py tests/test_gpu_bigshape.py -m gpu -x -q -k "not fused" > gpurun_out/pytest_nib.log 2>&1; echo "pytest nib rc=$?"; tail -2 gpurun_out/pytest_nib.log
for rep in 1 2; do
for envs in "" "MBU_HEAD_NIB=1"; do
  env $envs timeout 600 python bench.py --no-cpu --no-cudnn --no-e2e --no-extra --steps 20 --warmup 5 > gpurun_out/ab.json 2>gpurun_out/ab.err
  python - "${envs:-bytetab}" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
ks = {k["layer"]: k["ms"] for k in d["kernel_breakdown"]}
print(f'{sys.argv[1]:24s} value {d["value"]:7.1f} head {ks["head"]:.4f} upC4b {ks["up-C4.b"]:.4f}')
PY
done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:head_ -c 1 -o gpurun_out/prof_head_tab -f python tools/profile_forward.py --reps 1 > /dev/null 2>&1; echo "ncu tab rc=$?"
MBU_HEAD_NIB=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:head_ -c 1 -o gpurun_out/prof_head_nib -f python tools/profile_forward.py --reps 1 > /dev/null 2>&1; echo "ncu nib rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stem_tc -c 1 -o gpurun_out/prof_stem -f python tools/profile_forward.py --reps 1 > /dev/null 2>&1; echo "ncu stem rc=$?"
