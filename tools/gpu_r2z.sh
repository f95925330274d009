# round-2 final evidence: GPU tests, ncu launch list + DRAM traffic, two full captures, full bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_forward.py --reps 1 > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/traffic.csv python tools/profile_forward.py --reps 1 > gpurun_out/ncu_traffic.log 2>&1; echo "traffic rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 21 -c 1 -o gpurun_out/prof_stem2 -f python tools/profile_forward.py --reps 1 > /dev/null 2>&1; echo "full stem2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 40 -c 1 -o gpurun_out/prof_upc4a -f python tools/profile_forward.py --reps 1 > /dev/null 2>&1; echo "full upc4a rc=$?"
timeout 1500 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
