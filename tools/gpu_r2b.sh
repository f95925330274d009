mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_quantize.py -x -q > gpurun_out/pytest_q.log 2>&1; echo "q rc=$?"; tail -2 gpurun_out/pytest_q.log
bash tools/ab_bench.sh default build/ab/noexp.so build/ab/noepi.so 2>&1 | tee gpurun_out/ab.txt
MBU_LIB=build/ab/tl.so timeout 300 python tools/timeline_probe.py 2> gpurun_out/timeline.txt; echo "tl rc=$?"
