set -u
mkdir -p gpurun_out
python tools/peak_int8.py > gpurun_out/peak_int8.json 2>&1; cat gpurun_out/peak_int8.json
for s in 9 18 19; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc -s $s -c 1 \
  -o gpurun_out/prof_tc_$s -f python tools/profile_forward.py --reps 1 > gpurun_out/ncu_tc_$s.log 2>&1; echo "ncu $s rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stem -c 1 \
  -o gpurun_out/prof_stem -f python tools/profile_forward.py --reps 1 > gpurun_out/ncu_stem.log 2>&1; echo "ncu stem rc=$?"
