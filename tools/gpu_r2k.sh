mkdir -p gpurun_out
CUDA_LAUNCH_BLOCKING=1 timeout 900 python tools/layer_sweep.py 1024 2048 1 | grep -v '"ok"'; echo sweep done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
bash tools/ab_libs.sh build/ab/base.so build/ab/dual.so
