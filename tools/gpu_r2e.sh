mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
MBU_COL_SPLIT=1 timeout 900 python -m pytest tests/test_gpu_forward.py -x -q -k tiny > gpurun_out/pytest_cs.log 2>&1; echo "colsplit rc=$?"; tail -3 gpurun_out/pytest_cs.log
MBU_NBUF3=1 timeout 900 python -m pytest tests/test_gpu_forward.py -x -q -k tiny > gpurun_out/pytest_nb.log 2>&1; echo "nbuf3 rc=$?"; tail -3 gpurun_out/pytest_nb.log
bash tools/ab_env.sh "" 2>&1 | tee gpurun_out/ab_env.txt
