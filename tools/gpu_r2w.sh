timeout 1200 python -m pytest tests/test_gpu_forward.py tests/test_gpu_layers.py tests/test_gpu_bigshape.py -x -q 2>&1 | tail -2
bash tools/ab_libs.sh build/ab/base.so build/ab/lds128.so
