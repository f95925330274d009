mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 23 -c 1 -o gpurun_out/prof_dc1b -f python tools/profile_forward.py --reps 1 > /dev/null 2>&1; echo "full dc1b rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 25 -c 1 -o gpurun_out/prof_dc2b -f python tools/profile_forward.py --reps 1 > /dev/null 2>&1; echo "full dc2b rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 40 -c 1 -o gpurun_out/prof_upc4a -f python tools/profile_forward.py --reps 1 > /dev/null 2>&1; echo "full upc4a rc=$?"
