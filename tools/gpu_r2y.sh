mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 39 -c 1 -o gpurun_out/prof_upct4 -f python tools/profile_forward.py --reps 1 > /dev/null 2>&1; echo "full upct4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 30 -c 1 -o gpurun_out/prof_upct1 -f python tools/profile_forward.py --reps 1 > /dev/null 2>&1; echo "full upct1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stem_tc -s 1 -c 1 -o gpurun_out/prof_stem -f python tools/profile_forward.py --reps 1 > /dev/null 2>&1; echo "full stem rc=$?"
