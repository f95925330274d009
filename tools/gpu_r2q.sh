mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_forward.py tests/test_gpu_layers.py tests/test_gpu_bigshape.py tests/test_gpu_dp.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
bash tools/ab_libs.sh build/ab/base.so build/ab/head.so
