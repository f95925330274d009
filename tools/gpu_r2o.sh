mkdir -p gpurun_out
./tools/ubench_mma_sync > gpurun_out/ubench_mma_sync.txt 2>&1; cat gpurun_out/ubench_mma_sync.txt
./tools/ubench_tc > gpurun_out/ubench_tc.txt 2>&1; grep -E "mma_i8_ss" gpurun_out/ubench_tc.txt | head -8
./tools/ubench_fp4 > gpurun_out/ubench_fp4.txt 2>&1; grep -E '"mxf4_ss"' gpurun_out/ubench_fp4.txt
timeout 2400 python -m pytest tests/test_gpu_sanitizer.py -x -q -s > gpurun_out/pytest_san.log 2>&1; echo "san rc=$?"; grep -E "SUMMARY|passed|failed" gpurun_out/pytest_san.log | tail -8
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-cudnn --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d['config2_microbench']['rows']))"
