mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_bigshape.py -x -q > gpurun_out/pytest_big.log 2>&1; echo "big rc=$?"; tail -3 gpurun_out/pytest_big.log
timeout 1500 python -m pytest tests/test_gpu_conformance.py -x -q -s > gpurun_out/pytest_conf.log 2>&1; echo "conf rc=$?"; tail -5 gpurun_out/pytest_conf.log
MBU_LIB=build/ab/tl.so timeout 300 python tools/timeline_probe.py 2> gpurun_out/timeline.txt; echo "tl rc=$?"
