#!/bin/bash
# Quick GPU iteration: parity tests, a device-only bench line, the launch list.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu --no-cudnn ${BENCH_ARGS:-} > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_quick.json"))
print("value", round(d["value"], 1), "e2e", d["e2e"] and round(d["e2e"]["value"], 1), "ms", round(d["ms_per_step"], 3),
      "frac", round(d["roofline"]["frac"], 3))
for k in d["kernel_breakdown"]:
    print(f'{k["layer"]:12s} {k["ms"]:8.4f} {k["tops"]}')
PY
if [ "${LAUNCHES:-1}" = 1 ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python tools/profile_forward.py --reps 1 > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
fi
