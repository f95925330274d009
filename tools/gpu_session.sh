#!/bin/bash
# One gpurun session: GPU parity tests, the bench line, the launch list and an
# ncu --set full capture of the dominant kernel. Outputs land in gpurun_out/.
set -u
mkdir -p gpurun_out
OUT=gpurun_out
nvidia-smi > $OUT/nvidia_smi.txt 2>&1
cp MEASURED_PEAKS.json $OUT/ 2>/dev/null
lscpu > $OUT/lscpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
if [ "${SKIP_BENCH:-0}" != 1 ]; then
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cat $OUT/bench.json | head -c 3000; echo
fi
if [ "${SKIP_NCU:-0}" != 1 ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python tools/profile_forward.py --reps 1 > $OUT/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:conv_tc --csv --log-file $OUT/conv_traffic.csv python tools/profile_forward.py --reps 1 > $OUT/ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc -s ${NCU_SKIP:-2} -c ${NCU_COUNT:-3} \
  -o $OUT/prof_conv_tc -f python tools/profile_forward.py --reps 1 > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
