mkdir -p gpurun_out
for e in "" "MBU_MMA_WARPS=2"; do env $e CUDA_LAUNCH_BLOCKING=1 timeout 900 python tools/layer_sweep.py 1024 2048 1 | grep -v '"ok"'; echo "sweep [$e] done"; done
MBU_MMA_WARPS=2 timeout 900 python -m pytest tests/test_gpu_forward.py tests/test_gpu_layers.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu --no-cudnn --no-e2e --no-extra --steps 10 --warmup 5 > /dev/null 2>&1
for rep in 1 2; do
for e in "MBU_LIB=build/ab/base.so" "MBU_LIB=build/ab/dual5.so" "MBU_LIB=build/ab/dual5.so MBU_MMA_WARPS=2"; do
  env $e timeout 600 python bench.py --no-cpu --no-cudnn --no-e2e --no-extra --steps 20 --warmup 5 > gpurun_out/ab.json 2>gpurun_out/ab.err
  python - "$e" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
ks = {k["layer"]: k["ms"] for k in d["kernel_breakdown"]}
print(f'{sys.argv[1]:40s} value {d["value"]:7.1f}  ' + " ".join(f'{n}={v:.3f}' for n, v in ks.items()))
PY
done; done
