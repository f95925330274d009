mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
bash tools/ab_env.sh "" "MBU_NO_PRETEST=1" "MBU_NO_BIAS_REP=1" 2>&1 | tee gpurun_out/ab_env.txt
