mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_full.json"))
print("value", round(d["value"],1), "e2e", d["e2e"]["value"], "raster", d["e2e"]["raster_u8"]["value"], "frac", d["roofline"]["frac"])
print("cpu", d["cpu_baseline"]); print("numba", d["cpu_baseline_bitunet_numba"])
print("cudnn", {k: v for k, v in d["cudnn_fp16"].items() if k != "fused"}); print("fused", d["cudnn_fp16"].get("fused"))
print("c2", json.dumps(d["config2_microbench"])[:1500]); print("c5", json.dumps(d["config5_4k_latency"]))
print("clocks", d["clocks"])
PY
