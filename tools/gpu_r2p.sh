mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_sanitizer.py -q -s > gpurun_out/pytest_san.log 2>&1; echo "san rc=$?"; grep -E "SUMMARY|passed|failed|Barrier error" gpurun_out/pytest_san.log | sort | uniq -c | tail -8
timeout 900 python -m pytest tests/test_gpu_forward.py tests/test_gpu_layers.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
bash tools/ab_libs.sh build/ab/base.so build/ab/sf.so
