mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_forward.py tests/test_gpu_layers.py -x -q > gpurun_out/pytest_def.log 2>&1; echo "default pytest rc=$?"; tail -3 gpurun_out/pytest_def.log
MBU_NBUF3=1 MBU_COL_SPLIT=1 timeout 900 python -m pytest tests/test_gpu_forward.py tests/test_gpu_layers.py -x -q > gpurun_out/pytest_var.log 2>&1; echo "var pytest rc=$?"; tail -3 gpurun_out/pytest_var.log
bash tools/ab_env.sh "" "MBU_NBUF3=1" "MBU_COL_SPLIT=1" "MBU_NBUF3=1 MBU_COL_SPLIT=1" 2>&1 | tee gpurun_out/ab_env.txt
