mkdir -p gpurun_out
for e in "" "MBU_NO_BIAS_REP=1" "MBU_NO_PRETEST=1" "MBU_NO_BIAS_REP=1 MBU_NO_PRETEST=1"; do
  for r in 1 2 3; do
  env $e timeout 600 python -m pytest tests/test_gpu_forward.py -x -q -k "tiny" > gpurun_out/p.log 2>&1; echo "[$e] rep $r rc=$? $(tail -1 gpurun_out/p.log)"
  done
done
